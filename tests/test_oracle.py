"""Pins the CPU oracle (oracle/picard_oracle.c) before it is trusted as the checker.

(a) against the golden fixtures produced by the UNMODIFIED reference library
    (tests/golden/golden.json.gz, oracle/make_golden.py) — these travel to
    the GPU box where /root/reference does not exist;
(b) against the reference library itself (oracle/_ref) on fresh random
    cases when it is available;
(c) the glibc tanh restatement against this host's libm, bit for bit.
"""
import ctypes
import math

import numpy as np
import pytest

from oracle.oracle import ORC, REF
from tests.helpers import all_cases, load_golden, oracle_instance, oracle_policy

CASES = all_cases(load_golden())

LIBM = ctypes.CDLL("libm.so.6")
LIBM.tanh.restype = ctypes.c_double
LIBM.tanh.argtypes = [ctypes.c_double]


def _orc_tanh(x):
    if ORC.lib.orc_tanh_variant():
        return ORC.tanh(x)
    return ORC.lib.orc_tanh_nofma(x)


def test_tanh_matches_host_libm_bitwise():
    rng = np.random.default_rng(11)
    xs = np.concatenate([rng.uniform(-3, 3, 60000), rng.uniform(-30, 30, 20000),
                         rng.standard_normal(10000) * 1e-4,
                         10.0 ** rng.uniform(-300, 2, 10000) * rng.choice([-1, 1], 10000),
                         [0.0, -0.0, 1e-300, 22.0, -22.0, 0.34657359027997264, 1.0, -1.0,
                          math.inf, -math.inf]])
    bad = [x for x in xs if _orc_tanh(float(x)) != LIBM.tanh(float(x))]
    assert not bad, f"{len(bad)} mismatches, e.g. {bad[:3]}"


def test_tanh_golden_bits(golden):
    if not ORC.lib.orc_tanh_variant():
        pytest.skip("golden tanh bits were recorded on an FMA host")
    for xh, yh in golden["cases"]["tanh"]:
        assert ORC.tanh(float.fromhex(xh)) == float.fromhex(yh)


def test_expm1_nofma_matches_fdlibm_shape():
    # the SSE2 body cannot be reached through this host's IFUNC; check it
    # against the FMA body where both are exactly rounded-equal in practice
    rng = np.random.default_rng(3)
    for x in rng.uniform(-40, 40, 5000):
        a, b = ORC.lib.orc_expm1(float(x)), ORC.lib.orc_expm1_nofma(float(x))
        assert abs(a - b) <= 2 * abs(math.ulp(a))


def test_demand_and_apportion_known_answers(golden):
    # test_instance.cpp:28-54
    assert list(ORC.demand_counts(4, 8, 0.0)) == [2, 2, 2, 2]
    assert list(ORC.demand_counts(4, 120000, -1.0)) == [57600, 28800, 19200, 14400]
    assert list(ORC.apportion([3e6, 1e6], 80)) == [60, 20]
    assert list(ORC.apportion([1.0, 1.0, 1.0], 7)) == [3, 2, 2]
    for c in golden["cases"]["demand_counts"]:
        assert list(ORC.demand_counts(*c["args"])) == c["out"]
    for c in golden["cases"]["apportion"]:
        assert list(ORC.apportion(c["weights"], c["total"])) == c["out"]


def test_generate_instance_golden(golden):
    for c in golden["cases"]["generate_instance"]:
        d = ORC.generate_instance_arrays(*c["args"], geometry=c.get("geometry", 0))
        assert d["product"].tolist() == c["product"]
        assert d["reward_row"].tolist() == c["origin"]
        assert [float(x).hex() for x in d["reward_table"]] == c["reward_table"]
        assert d["capacity"].tolist() == c["capacity"]
        assert d["inventory"].tolist() == c["inventory"]


def test_partition_known_answers(golden):
    c = golden["cases"]["product_hand_trace"]
    hand = oracle_instance(dict(kind="explicit", nodes=1, products=4, capacity=[10], inventory=[0, 0, 0, 0],
                                product=[0, 0, 0, 0, 1, 1, 1, 2, 2, 3], reward_row=list(range(10)),
                                reward_table=[1.0] * 10), ORC)
    owner = ORC.product_partition(hand, 2, 3)
    assert owner.tolist() == c["owner_m2"]
    # test_instance.cpp:231-240: {p0,p3} vs {p1,p2}, loads 5/5
    assert owner[9] == owner[0] and owner[4] == 1 - owner[0] and owner[7] == 1 - owner[0]
    assert int((owner == 0).sum()) == 5
    assert ORC.product_partition(hand, 1, 3).tolist() == c["owner_m1"]
    counts = np.bincount(ORC.uniform_partition(10000, 10, 1234), minlength=10)
    assert counts.tolist() == golden["cases"]["uniform_partition"]["counts"]
    assert all(abs(int(x) - 1000) <= 120 for x in counts)


@pytest.mark.parametrize("name,case", CASES, ids=[n for n, _ in CASES])
def test_oracle_matches_reference_golden(name, case):
    inst = oracle_instance(case["instance"], ORC)
    pol = oracle_policy(case["policy"], inst, ORC)
    seq, evals = ORC.sequential(inst, pol)
    assert seq.tolist() == case["sequential"]
    assert evals == inst.horizon
    init = None if case["initial_cache"] is None else np.array(case["initial_cache"], np.int32)
    r = ORC.picard(inst, pol, np.array(case["owner"], np.int32), case["processes"],
                   max_steps=case["config"]["max_steps"], record_trace=True, reference=seq,
                   history=case["history"] is not None, initial_cache=init)
    assert r.actions.tolist() == case["actions"]
    assert r.actions.tolist() == case["sequential"]  # Prop. 1
    assert r.iterations_to_converged == case["iterations_to_converged"]
    assert r.iterations_to_correct == case["iterations_to_correct"]
    assert r.conflicts == case["conflicts"]
    assert r.policy_eval_count_sequential_equivalent == case["seq_equiv"]
    assert r.total_policy_evals == case["total_evals"]
    assert [list(x) for x in r.trace] == case["trace"]
    if case["history"] is not None:
        assert r.history.tolist() == case["history"]
    assert ORC.total_reward(inst, r.actions) == case["total_reward"]


def test_toy_hand_trace(golden):
    # test_engine.cpp:100-138 — the hand-traced expectations themselves
    c = golden["cases"]["toy_two_order"]
    assert c["sequential"] == [0, 1]
    assert c["iterate_once_1"] == dict(cache=[0, 0], evals=[1, 1], changed=[0, 1])
    assert c["iterate_once_2"]["cache"] == [0, 1]
    assert c["iterations_to_correct"] == 2 and c["conflicts"] == 1
    inst = oracle_instance(c["instance"], ORC)
    g = oracle_policy(dict(kind=0, gamma=0.0), inst, ORC)
    cache, evals, changed = ORC.iterate_once(inst, g, np.array([0, 1], np.int32), 2, np.array([-1, -1]), 0, 2)
    assert cache.tolist() == [0, 0] and evals.tolist() == [1, 1] and changed.tolist() == [0, 1]
    # single process: correct after 1, converged after 2, 2T evaluations (:81-98)
    s = golden["cases"]["toy_single_process"]
    assert s["iterations_to_correct"] == 1 and s["iterations_to_converged"] == 2
    assert s["seq_equiv"] == 4 and s["total_evals"] == 4
    # infeasible cache degrades to declining (:140-173)
    assert golden["cases"]["infeasible_cache"]["actions"] == [0, -1, -1]


def test_textbook_fixed_point_equals_engine_iterates(golden):
    # test_engine.cpp:229-299: naive Algorithm 1 == the engine's per-iteration caches
    for case in golden["cases"]["textbook_grid"]:
        inst = oracle_instance(case["instance"], ORC)
        pol = oracle_policy(case["policy"], inst, ORC)
        hist = ORC.naive_fixed_point(inst, pol, np.array(case["owner"], np.int32), case["processes"])
        assert hist.tolist() == case["history"]
        assert len(hist) == case["iterations_to_converged"]


def test_dual_forward_golden(golden):
    c = golden["cases"]["dual_forward"]
    from types import SimpleNamespace as NS
    p = NS(kind=2, hidden=64, gamma=0.0, horizon=c["horizon"])
    p.w1, p.b1, p.w2, p.b2, p.w3, p.b3 = ORC.seeded_mlp(7, 6, c["seed"])
    prices = ORC.mlp_forward(p, c["features"])
    if ORC.lib.orc_tanh_variant():
        assert [float(x).hex() for x in prices] == c["prices"]
    inst = oracle_instance(dict(kind="explicit", nodes=3, products=1, capacity=c["init_capacity"],
                                inventory=c["init_inventory"], product=[0] * 10, reward_row=[0] * 10,
                                reward_table=c["rewards"]), ORC)
    a = ORC.policy_evaluate(inst, p, np.array(c["state_capacity"], np.int32),
                            np.array(c["state_inventory"], np.int32), c["t"])
    assert a == c["action"]


@pytest.mark.skipif(REF is None, reason="reference library not built here")
def test_oracle_matches_reference_library_random():
    from types import SimpleNamespace as NS
    rng = np.random.default_rng(5)
    for seed in range(1000, 1030):
        J, I, T, beta, cov, s = ORC.small_random_params(seed)
        assert (J, I, T, beta, cov, s) == REF.small_random_params(seed)
        inst = NS(**ORC.generate_instance_arrays(J, I, T, beta, cov, s))
        M = int(rng.integers(1, 10))
        owner = ORC.uniform_partition(T, M, seed) if seed % 3 else ORC.product_partition(inst, M, seed)
        for kind in (0, 1, 2):
            p = NS(kind=kind, hidden=64, gamma=float(rng.uniform(0, 3)), horizon=None)
            if kind == 2:
                p.w1, p.b1, p.w2, p.b2, p.w3, p.b3 = ORC.seeded_mlp(2 * J + 1, 2 * J, seed)
            ms = int(rng.integers(0, 7))
            seq_r, _ = REF.sequential(inst, p)
            a = REF.picard(inst, p, owner, M, max_steps=ms, record_trace=True, reference=seq_r, history=True)
            b = ORC.picard(inst, p, owner, M, max_steps=ms, record_trace=True, reference=seq_r, history=True)
            assert np.array_equal(a.actions, b.actions) and a.trace == b.trace
            assert np.array_equal(a.history, b.history)
            assert (a.conflicts, a.iterations_to_correct) == (b.conflicts, b.iterations_to_correct)


@pytest.mark.skipif(REF is None, reason="reference library not built here")
def test_oracle_matches_reference_library_j100_dual():
    from types import SimpleNamespace as NS
    inst = NS(**ORC.generate_instance_arrays(100, 30, 3000, 0.0, 0.8, 7, geometry=1))
    p = NS(kind=2, hidden=64, gamma=0.0, horizon=None)
    p.w1, p.b1, p.w2, p.b2, p.w3, p.b3 = ORC.seeded_mlp(201, 200, 5)
    owner = ORC.product_partition(inst, 64, 1)
    seq_r, _ = REF.sequential(inst, p)
    seq_o, _ = ORC.sequential(inst, p)
    assert np.array_equal(seq_r, seq_o)
    a = REF.picard(inst, p, owner, 64, record_trace=True, reference=seq_r)
    b = ORC.picard(inst, p, owner, 64, record_trace=True, reference=seq_r)
    assert np.array_equal(a.actions, b.actions) and a.trace == b.trace
