"""CPU-side tests of the product library: the C ABI loads and exports every
declared symbol, the host-side serial-RNG inputs reproduce the oracle (and
hence the reference) bit for bit, and errors map onto the reference's
exception types. No compute entry point is called without a GPU."""
import os
import re

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from paper_2406_01939_b200 import _capi
from oracle.oracle import ORC
from tests.helpers import is_run_partition, oracle_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "picard_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcd_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(_capi.LIB, s), s
    # and the ctypes binding covers the whole header
    assert set(syms) == set(_capi.SIGNATURES), set(syms) ^ set(_capi.SIGNATURES)


def test_library_is_sm100a():
    so = _capi.LIB_PATH
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    assert "sm_100a" in out, out


@pytest.mark.parametrize("args", [(5, 40, 1000, -0.6, 0.8, 1), (30, 10000, 30000, 0.0, 0.8, 7),
                                  (1, 10, 10000, 0.0, 0.8, 7), (3, 20, 200, 0.0, 0.8, 5),
                                  (12, 7, 999, -1.3, 0.55, 12345)])
def test_generate_instance_matches_oracle(args):
    a = P.generate_instance(*args)
    b = ORC.generate_instance_arrays(*args)
    assert np.array_equal(a.product, b["product"])
    assert np.array_equal(a.reward_row, b["reward_row"])
    assert np.array_equal(a.reward_table.ravel(), b["reward_table"])
    assert np.array_equal(a.capacity, b["capacity"])
    assert np.array_equal(a.inventory.ravel(), b["inventory"])


def test_generate_instance_j100_geometry_matches_oracle():
    a = P.generate_instance(100, 1000, 100000, 0.0, 0.8, 7)
    b = ORC.generate_instance_arrays(100, 1000, 100000, 0.0, 0.8, 7, geometry=1)
    for k in ("product", "reward_row", "capacity"):
        assert np.array_equal(getattr(a, k), b[k]), k
    assert np.array_equal(a.inventory.ravel(), b["inventory"])
    assert np.array_equal(a.reward_table.ravel(), b["reward_table"])


def test_generate_instance_rejects_bad_parameters():
    # test_instance.cpp:138-146
    for args in [(0, 10, 10, 0.0), (31, 10, 10, 0.0), (5, 0, 10, 0.0), (5, 10, 0, 0.0), (5, 10, 10, 0.5),
                 (5, 10, 10, 0.0, 0.0), (5, 10, 10, 0.0, 1.5)]:
        kw = dict(geometry=0)
        with pytest.raises(P.InvalidArgument):
            P.generate_instance(*args, **kw)


def test_generated_instance_sizing_identities():
    # test_instance.cpp:80-117
    for seed in (1, 9, 77):
        inst = P.generate_instance(5, 40, 1000, -0.6, 0.8, seed)
        counts = ORC.demand_counts(40, 1000, -0.6)
        assert int(inst.capacity.sum()) == round(0.8 * 1000)
        assert np.array_equal(np.bincount(inst.product, minlength=40), counts)
        assert np.array_equal(inst.inventory.sum(1), np.round(0.8 * counts).astype(int))
        r = inst.reward_table[inst.reward_row]
        assert (r >= 0).all() and (r <= 1).all()
        assert (r[np.arange(inst.horizon), inst.origin] == 1.0).all()


@pytest.mark.parametrize("M,seed", [(1, 3), (2, 3), (7, 99), (64, 1), (5000, 4)])
def test_product_partition_matches_oracle(M, seed):
    inst = P.generate_instance(4, 60, 700, -0.9, 0.8, 13)
    plan = P.make_product_partition(inst, M, seed)
    assert np.array_equal(plan.owner, ORC.product_partition(inst, M, seed))
    # each product on one process (test_instance.cpp:243-255)
    for p in range(60):
        assert len(set(plan.owner[inst.product == p].tolist())) <= 1


@pytest.mark.parametrize("J,I,T,M", [(4, 60, 700, 64), (4, 60, 700, 200), (10, 300, 20000, 4096), (3, 5, 40, 1000),
                                     (4, 60, 700, 7)])
def test_product_chunk_partition_is_a_balanced_run_partition(J, I, T, M):
    inst = P.generate_instance(J, I, T, -0.5, 0.8, 13)
    plan = P.make_product_chunk_partition(inst, M)
    assert plan.owner.min() >= 0 and plan.owner.max() < M
    assert is_run_partition(plan.owner, inst.product)
    q = np.bincount(inst.product, minlength=I)
    used = int((q > 0).sum())
    if M < used:  # falls back to the reference's product partition
        assert np.array_equal(plan.owner, P.make_product_partition(inst, M, 1).owner)
        return
    loads = np.bincount(plan.owner, minlength=M)
    L = int(loads.max())
    # L is the smallest chunk length that fits in M processes
    assert int(np.ceil(q / L).sum()) <= M
    if L > 1:
        assert int(np.ceil(q / (L - 1)).sum()) > M
    # chunks of a product differ by at most one order and follow time order
    for p in range(I):
        own = plan.owner[inst.product == p]
        if own.size:
            assert (np.diff(own) >= 0).all()
            c = np.bincount(own - own.min())
            c = c[c > 0]
            assert c.max() - c.min() <= 1
def _window_cuts(times, W, L):
    """Greedy restatement: a chunk grows while no W-long interval holds more
    than L of its orders (tested at each new order)."""
    cuts, k0, j = [0], 0, 0
    for k in range(len(times)):
        while times[j] <= times[k] - W:
            j += 1
        if k - max(k0, j) + 1 > L:
            k0 = k
            cuts.append(k)
    return cuts


@pytest.mark.parametrize("J,I,T,M,W", [(5, 20, 3000, 64, 300), (5, 20, 3000, 200, 100), (8, 50, 5000, 30, 500),
                                       (3, 7, 2000, 5, 0), (4, 12, 1500, 40, 1500), (6, 30, 4000, 97, 257)])
def test_product_window_partition_bounds_every_window(J, I, T, M, W):
    inst = P.generate_instance(J, I, T, -0.5, 0.8, 13)
    plan = P.make_product_window_partition(inst, M, W)
    assert plan.processes == M and plan.owner.min() >= 0 and plan.owner.max() < M
    assert is_run_partition(plan.owner, inst.product)
    q = np.bincount(inst.product, minlength=I)
    used = int((q > 0).sum())
    if M < used:  # falls back to the reference's product partition
        assert np.array_equal(plan.owner, P.make_product_partition(inst, M, 1).owner)
        return
    Wn = T if W <= 0 or W > T else W
    times = [np.flatnonzero(inst.product == p) for p in range(I)]
    # the bound: the largest count of one process's orders in any Wn-interval
    L = 0
    for p in range(I):
        for proc in np.unique(plan.owner[times[p]]):
            ts = np.flatnonzero(plan.owner == proc)
            L = max(L, int((np.searchsorted(ts, ts + Wn) - np.arange(ts.size)).max()))
    # same cuts as the greedy restatement at L, and L is minimal for M chunks
    for p in range(I):
        own = plan.owner[times[p]]
        if own.size:
            assert (np.diff(own) >= 0).all()
            assert list(np.flatnonzero(np.diff(own)) + 1) == _window_cuts(times[p], Wn, L)[1:]
    assert sum(len(_window_cuts(t, Wn, L)) for t in times if t.size) <= M
    if L > 1:
        assert sum(len(_window_cuts(t, Wn, L - 1)) for t in times if t.size) > M


def test_product_window_partition_rejects_bad_input():
    inst = P.generate_instance(3, 5, 100, 0.0, 0.8, 1)
    with pytest.raises(P.InvalidArgument):
        P.make_product_window_partition(inst, 0, 10)




def test_product_partition_hand_trace(golden):
    c = golden["cases"]["product_hand_trace"]
    inst = P.Instance(1, 4, 10, [0, 0, 0, 0, 1, 1, 1, 2, 2, 3], list(range(10)), [[1.0]] * 10, [10], [[0]] * 4)
    assert P.make_product_partition(inst, 2, 3).owner.tolist() == c["owner_m2"]
    assert P.make_product_partition(inst, 1, 3).owner.tolist() == c["owner_m1"]


def test_uniform_partition_matches_oracle_and_balance(golden):
    plan = P.make_uniform_time_partition(10000, 10, 1234)
    assert np.array_equal(plan.owner, ORC.uniform_partition(10000, 10, 1234))
    assert np.bincount(plan.owner, minlength=10).tolist() == golden["cases"]["uniform_partition"]["counts"]
    assert P.make_uniform_time_partition(4, 1, 3).owner.tolist() == [0, 0, 0, 0]
    assert P.make_uniform_time_partition(0, 5, 3).owner.size == 0
    with pytest.raises(P.ContractViolation):
        P.make_uniform_time_partition(10, 0, 1)


def test_seeded_mlp_matches_oracle_and_roundtrips(tmp_path):
    p = P.MlpParams.seeded_uniform(7, 6, 12345)
    ref = ORC.seeded_mlp(7, 6, 12345)
    for a, b in zip((p.w1, p.b1, p.w2, p.b2, p.w3, p.b3), ref):
        assert np.array_equal(a, b)
    assert all(np.abs(x).max() < 0.1 for x in (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3))
    path = str(tmp_path / "params.bin")
    p.save(path)
    q = P.MlpParams.load(path)
    assert q.widths == p.widths and all(np.array_equal(a, b) for a, b in zip(
        (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3), (q.w1, q.b1, q.w2, q.b2, q.w3, q.b3)))
    os.truncate(path, 64)  # test_policies.cpp:332-344
    with pytest.raises(RuntimeError):
        P.MlpParams.load(path)
    assert P.MlpParams.zeros(5, 4).all_zero()


def test_total_reward_and_compare(golden):
    toy = P.Instance(2, 1, 2, [0, 0], [0, 1], [[0.9, 0.1], [0.8, 0.2]], [1, 1], [[1, 1]])
    assert abs(P.fo_total_reward(toy, [0, 1]) - 1.1) < 1e-12  # test_fo_env.cpp:67-71
    assert P.fo_total_reward(toy, [-1, -1]) == 0.0
    a = [0, 1, -1, 1]
    assert P.compare_to_oracle(a, a) == (True, None)
    assert P.compare_to_oracle(a, [0, 1, -1, 0]) == (False, 3)  # test_engine.cpp:563-582
    with pytest.raises(P.ContractViolation):
        P.compare_to_oracle(a, a[:3])
    for c in golden["cases"]["oracle_grid"][:10]:
        inst = P.Instance(**{k: v for k, v in vars(oracle_instance(c["instance"], ORC)).items()})
        assert P.fo_total_reward(inst, c["actions"]) == c["total_reward"]


def test_shard_processes_is_balanced():
    inst = P.generate_instance(10, 1000, 100000, 0.0, 0.8, 7)
    plan = P.make_product_partition(inst, 4096, 1)
    for ranks in (1, 2, 4, 8):
        r = P.shard_processes(plan, ranks)
        assert r.min() >= 0 and r.max() < ranks
        loads = np.bincount(plan.owner, minlength=plan.processes)
        per = np.bincount(r, weights=loads, minlength=ranks)
        assert per.max() - per.min() <= loads.max()


def test_device_entry_points_fail_loudly_without_gpu():
    if P.device_count() > 0:
        pytest.skip("a GPU is visible")
    inst = P.generate_instance(3, 5, 50, 0.0, 0.8, 1)
    with pytest.raises(P.CudaError, match="no CPU fallback"):
        P.picard_simulate(inst, P.GreedyPolicy(), P.make_product_partition(inst, 2, 1))


def test_dual_policy_rejects_wrong_widths():
    with pytest.raises(P.ContractViolation):
        P.DualNetworkPolicy(P.MlpParams.zeros(7, 5), nodes=3)


def test_c3_instance_and_policy_equal_the_reference_generator():
    """The bench workload's inputs (C3 with the J>30 synthetic geometry) are
    bit-identical to the compiled reference's generate_instance /
    MlpParams::seeded_uniform (instance.cpp:80-140, mlp.cpp:117-129)."""
    import numpy as np
    import pytest
    from oracle.oracle import REF
    if REF is None:
        pytest.skip("oracle/_ref not built")
    import paper_2406_01939_b200 as P
    J, I, T = 100, 10_000, 10_000_000
    ref = REF.generate_instance_arrays(J, I, T, 0.0, 0.8, 7, geometry=1)
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    assert np.array_equal(inst.product, ref["product"])
    assert np.array_equal(inst.reward_row, ref["reward_row"])
    assert np.array_equal(inst.reward_table.ravel(), ref["reward_table"])
    assert np.array_equal(inst.capacity, ref["capacity"])
    assert np.array_equal(inst.inventory.ravel(), ref["inventory"])
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    for a, b in zip((pol.w1, pol.b1, pol.w2, pol.b2, pol.w3, pol.b3), REF.seeded_mlp(2 * J + 1, 2 * J, 5)):
        assert np.array_equal(a, b)
