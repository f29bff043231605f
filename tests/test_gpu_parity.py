"""GPU parity tests proper: the sm_100a engine (through the C ABI) against the
oracle and the reference's golden fixtures. Integer outputs (actions,
iteration counts, conflicts, evaluation counters, trace rows, per-iteration
caches) must be bit-exact; total reward is compared with rel. tol 1e-12
(north_star allows 1e-4; the engine is exact so we hold it far tighter)."""
from types import SimpleNamespace as NS

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import ORC, OracleError
from tests.helpers import (all_cases, is_run_partition, load_golden, oracle_instance, oracle_policy, product_instance,
                           product_policy)

pytestmark = pytest.mark.gpu

CASES = all_cases(load_golden())


def run_gpu(case, engine="auto", history=True):
    ons = oracle_instance(case["instance"], ORC)
    inst = product_instance(ons)
    pol = product_policy(case["policy"], inst)
    plan = P.PartitionPlan(case["processes"], case["owner"])
    cfg = P.PicardConfig(max_steps=case["config"]["max_steps"], record_trace=True, engine=engine)
    init = case["initial_cache"]
    with P.Simulator(inst, pol) as sim:
        sim.set_plan(plan)
        r = sim.simulate(cfg, init, case["sequential"], record_history=history)
    return inst, r


def check(case, r):
    assert r.actions.tolist() == case["actions"]
    assert r.iterations_to_converged == case["iterations_to_converged"]
    assert r.iterations_to_correct == case["iterations_to_correct"]
    assert r.conflicts == case["conflicts"]
    assert r.policy_eval_count_sequential_equivalent == case["seq_equiv"]
    assert r.total_policy_evals == case["total_evals"]
    assert [list(x.astuple()) for x in r.trace] == case["trace"]
    if case.get("history") is not None:
        assert r.history.tolist() == case["history"]


@pytest.mark.parametrize("name,case", CASES, ids=[n for n, _ in CASES])
def test_engine_matches_reference_golden(name, case):
    inst, r = run_gpu(case, "auto")
    check(case, r)
    assert abs(P.fo_total_reward(inst, r.actions) - case["total_reward"]) <= 1e-12 * max(1.0, abs(case["total_reward"]))


@pytest.mark.parametrize("name,case", CASES[::3], ids=[n for n, _ in CASES[::3]])
def test_replay_engine_matches_reference_golden(name, case):
    _, r = run_gpu(case, "replay")
    check(case, r)


@pytest.mark.parametrize("name,case", CASES, ids=[n for n, _ in CASES])
def test_general_engine_matches_reference_golden(name, case):
    """The general closed form (any plan, any cache) on every golden case,
    run partitions included."""
    _, r = run_gpu(case, "general")
    check(case, r)
    assert r.timing["engine_used"] == 4


def test_auto_engine_choice(golden):
    """AUTO: run partitions take the run-partition closed form, every other
    plan the general closed form."""
    for name, case in CASES[::4]:
        owner = np.array(case["owner"])
        prod = oracle_instance(case["instance"], ORC).product
        _, r = run_gpu(case, "auto", history=False)
        assert r.timing["engine_used"] == (2 if is_run_partition(owner, prod) else 4), name


def test_product_engine_is_used_for_product_partitions(golden):
    """engine=PRODUCT on every golden case: run partitions (product partitions
    and any plan whose per-product stretches qualify) give the golden result,
    the others are refused with InvalidArgument."""
    used = 0
    for name, case in CASES:
        owner = np.array(case["owner"])
        prod = oracle_instance(case["instance"], ORC).product
        if not is_run_partition(owner, prod):
            with pytest.raises(P.InvalidArgument):
                run_gpu(case, "product", history=False)
            continue
        _, r = run_gpu(case, "product")
        check(case, r)
        assert r.timing["engine_used"] == 2
        used += 1
    assert used >= 20


def test_create_refuses_out_of_range_orders():
    """pcd_create checks every order's product and reward row on the device and
    reports the first offending time step (a product before a reward row at
    the same step), like the reference's instance validation."""
    base = P.generate_instance(4, 6, 200, 0.0, 0.8, 3)
    pol = P.GreedyPolicy()

    def inst(prod, rrow):
        return P.Instance(base.nodes, base.products, base.horizon, prod, rrow, base.reward_table, base.capacity,
                          base.inventory)
    prod, rrow = np.array(base.product), np.array(base.reward_row)
    p2 = prod.copy(); p2[57] = base.products
    r2 = rrow.copy(); r2[31] = np.asarray(base.reward_table).shape[0]
    for pr, rr, msg in ((p2, rrow, "order product out of range at t=57"), (prod, r2, "reward row out of range at t=31"),
                        (p2, r2, "reward row out of range at t=31")):
        with pytest.raises(P.InvalidArgument, match=msg):
            P.Simulator(inst(pr, rr), pol)
    with P.Simulator(inst(prod, rrow), pol):
        pass


def test_toy_iterate_once_hand_trace(golden):
    # test_engine.cpp:100-138
    toy = P.Instance(2, 1, 2, [0, 0], [0, 1], [[0.9, 0.1], [0.8, 0.2]], [1, 1], [[1, 1]])
    plan = P.PartitionPlan(2, [0, 1])
    cache = np.full(2, -1, np.int32)
    out = P.picard_iterate_once(toy, P.GreedyPolicy(), plan, cache, 0, 2)
    assert cache.tolist() == [0, 0]
    assert out.changed_slots.tolist() == [0, 1]
    assert out.evals_per_process.tolist() == [1, 1]
    P.picard_iterate_once(toy, P.GreedyPolicy(), plan, cache, 0, 2)
    assert cache.tolist() == [0, 1]
    assert P.sequential_simulate(toy, P.GreedyPolicy()).actions.tolist() == [0, 1]


@pytest.mark.parametrize("engine", ["replay", "auto", "general"])
def test_iterate_once_random_caches_match_oracle(engine):
    """Arbitrary (even garbage) caches, windows and checkpoints: one iteration
    must reproduce picard_iterate_once exactly (engine.hpp:358-444)."""
    rng = np.random.default_rng(17)
    for seed in range(40):
        J, I, T, beta, cov, s = ORC.small_random_params(700 + seed)
        ons = NS(**ORC.generate_instance_arrays(J, I, T, beta, cov, s))
        inst = product_instance(ons)
        M = int(rng.integers(1, 6))
        owner = ORC.product_partition(ons, M, seed) if seed % 2 == 0 else ORC.uniform_partition(T, M, seed)
        kind = seed % 3
        spec = dict(kind=kind, gamma=1.3, seed=seed)
        opol = oracle_policy(spec, ons, ORC)
        pol = product_policy(spec, inst)
        cache = rng.integers(-3, J + 2, T).astype(np.int32)
        lo = int(rng.integers(0, T))
        hi = int(rng.integers(lo, T + 1))
        # a feasible checkpoint: the state after a random feasible prefix
        ck_cap = ons.capacity.copy()
        ck_inv = ons.inventory.copy().reshape(I, J)
        for t in range(lo):
            a = int(rng.integers(-1, J))
            p = ons.product[t]
            if a >= 0 and ck_cap[a] > 0 and ck_inv[p, a] > 0:
                ck_cap[a] -= 1
                ck_inv[p, a] -= 1
        want, want_evals, want_changed = ORC.iterate_once(ons, opol, owner, M, cache, lo, hi, ck_cap, ck_inv.ravel())
        got = cache.copy()
        out = P.picard_iterate_once(inst, pol, P.PartitionPlan(M, owner), got, lo, hi, ck_cap, ck_inv, engine)
        assert got.tolist() == want.tolist(), (seed, engine)
        assert out.evals_per_process.tolist() == want_evals.tolist()
        assert out.changed_slots.tolist() == want_changed.tolist()


def _dual_case(J, I, T, M, part, seed=7, theta=5, max_steps=0):
    ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, seed, geometry=0 if J <= 30 else 1))
    inst = product_instance(ons)
    owner = ORC.product_partition(ons, M, 1) if part == "product" else ORC.uniform_partition(T, M, 1)
    spec = dict(kind=2, gamma=0.0, seed=theta)
    return ons, inst, owner, oracle_policy(spec, ons, ORC), product_policy(spec, inst)


@pytest.mark.parametrize("J,I,T,M,part", [(10, 300, 20000, 512, "product"), (30, 200, 12000, 256, "product"),
                                          (100, 40, 4000, 64, "product"), (10, 100, 6000, 64, "uniform"),
                                          (1, 10, 10000, 16, "product")])
def test_dual_policy_matches_oracle_counters(J, I, T, M, part):
    ons, inst, owner, opol, pol = _dual_case(J, I, T, M, part)
    seq, _ = ORC.sequential(ons, opol)
    want = ORC.picard(ons, opol, owner, M, record_trace=True, reference=seq)
    r = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(record_trace=True),
                          reference_actions=seq)
    assert r.actions.tolist() == seq.tolist()
    assert r.iterations_to_converged == want.iterations_to_converged
    assert r.iterations_to_correct == want.iterations_to_correct
    assert r.conflicts == want.conflicts
    assert r.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent
    assert r.total_policy_evals == want.total_policy_evals
    assert [x.astuple() for x in r.trace] == [tuple(x) for x in want.trace]


def _chunk_case(J, I, T, M, kind, seed=7):
    ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, seed, geometry=0 if J <= 30 else 1))
    inst = product_instance(ons)
    owner = P.make_product_chunk_partition(inst, M).owner
    spec = dict(kind=kind, gamma=1.7, seed=5)
    return ons, inst, owner, oracle_policy(spec, ons, ORC), product_policy(spec, inst)


def _same_run(r, want, seq):
    assert r.actions.tolist() == seq.tolist()
    assert r.iterations_to_converged == want.iterations_to_converged
    assert r.iterations_to_correct == want.iterations_to_correct
    assert r.conflicts == want.conflicts
    assert r.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent
    assert r.total_policy_evals == want.total_policy_evals
    assert [x.astuple() for x in r.trace] == [tuple(x) for x in want.trace]


@pytest.mark.parametrize("J,I,T,M,kind", [(10, 300, 20000, 1500, 2), (30, 50, 6000, 400, 2), (100, 20, 3000, 120, 2),
                                          (10, 100, 8000, 500, 0), (10, 100, 8000, 500, 1), (1, 10, 10000, 64, 2),
                                          (100, 40, 4000, 300, 2)])
def test_chunk_partition_matches_oracle(J, I, T, M, kind):
    """Product chunks (several processes per product, contiguous stretches):
    the closed form starts every stretch from the frozen-cache replay state
    (k_xinit); trajectory and every per-iteration counter as the oracle."""
    ons, inst, owner, opol, pol = _chunk_case(J, I, T, M, kind)
    assert len(np.unique(owner)) > I  # products really are split
    seq, _ = ORC.sequential(ons, opol)
    want = ORC.picard(ons, opol, owner, M, record_trace=True, reference=seq)
    for engine in (("product", "product_fp64") if kind == 2 else ("product",)):
        r = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(record_trace=True, engine=engine),
                              reference_actions=seq)
        assert r.timing["tc_used"] == (1 if engine == "product" and kind == 2 else 0)
        _same_run(r, want, seq)


def test_chunk_partition_windows_and_warm_starts_match_oracle():
    ons, inst, owner, opol, pol = _chunk_case(10, 50, 3000, 160, 2)
    seq, _ = ORC.sequential(ons, opol)
    draft, _ = ORC.sequential(ons, NS(kind=1, hidden=64, gamma=2.0, horizon=None))
    for ms in (1, 7, 300, 0):
        for init in (None, draft):
            want = ORC.picard(ons, opol, owner, 160, max_steps=ms, record_trace=True, reference=seq,
                              initial_cache=init)
            for engine in ("product", "product_fp64"):
                r = P.picard_simulate(inst, pol, P.PartitionPlan(160, owner),
                                      P.PicardConfig(max_steps=ms, record_trace=True, engine=engine), init, seq)
                _same_run(r, want, seq)


@pytest.mark.parametrize("engine", ["product", "product_fp64"])
def test_chunk_partition_iterate_once_random_caches_match_oracle(engine):
    """Arbitrary caches, windows and checkpoints under product chunks and mixed
    run plans (whole products + chunks): one iteration equals
    picard_iterate_once exactly — the closed form holds for any cache."""
    rng = np.random.default_rng(23)
    for seed in range(30):
        J, I, T, beta, cov, s = ORC.small_random_params(900 + seed)
        ons = NS(**ORC.generate_instance_arrays(J, I, T, beta, cov, s))
        inst = product_instance(ons)
        M = int(rng.integers(I, 4 * I + 8))
        owner = P.make_product_chunk_partition(inst, M).owner.copy()
        if seed % 2:  # mixed: merge some whole products onto one process
            q = np.bincount(ons.product, minlength=I)
            whole = [p for p in range(I) if q[p] and len(np.unique(owner[ons.product == p])) == 1]
            for p in whole[1::2]:
                owner[ons.product == p] = owner[ons.product == whole[0]][0]
        kind = 2 if engine == "product" else seed % 3
        spec = dict(kind=kind, gamma=1.3, seed=seed)
        opol = oracle_policy(spec, ons, ORC)
        pol = product_policy(spec, inst)
        cache = rng.integers(-3, J + 2, T).astype(np.int32)
        lo = int(rng.integers(0, T))
        hi = int(rng.integers(lo, T + 1))
        ck_cap = ons.capacity.copy()
        ck_inv = ons.inventory.copy().reshape(I, J)
        for t in range(lo):
            a = int(rng.integers(-1, J))
            p = ons.product[t]
            if a >= 0 and ck_cap[a] > 0 and ck_inv[p, a] > 0:
                ck_cap[a] -= 1
                ck_inv[p, a] -= 1
        want, want_evals, want_changed = ORC.iterate_once(ons, opol, owner, M, cache, lo, hi, ck_cap, ck_inv.ravel())
        got = cache.copy()
        out = P.picard_iterate_once(inst, pol, P.PartitionPlan(M, owner), got, lo, hi, ck_cap, ck_inv, engine)
        assert got.tolist() == want.tolist(), seed
        assert out.evals_per_process.tolist() == want_evals.tolist()
        assert out.changed_slots.tolist() == want_changed.tolist()


@pytest.mark.parametrize("tiles", [1, 3])
def test_tensor_core_work_list_pulls_match(tiles):
    """Fewer CTAs than processes / 128: rows pull processes from the work list
    mid-iteration (per-process counters flushed at each switch)."""
    ons, inst, owner, opol, pol = _chunk_case(30, 100, 20000, 900, 2)
    seq, _ = ORC.sequential(ons, opol)
    ref = P.picard_simulate(inst, pol, P.PartitionPlan(900, owner),
                            P.PicardConfig(record_trace=True, engine="product_fp64"), reference_actions=seq)
    r = P.picard_simulate(inst, pol, P.PartitionPlan(900, owner),
                          P.PicardConfig(record_trace=True, engine="product", tc_tiles=tiles), reference_actions=seq)
    assert r.timing["tc_used"] == 1
    assert r.actions.tolist() == seq.tolist()
    assert [x.astuple() for x in r.trace] == [x.astuple() for x in ref.trace]
    assert (r.conflicts, r.iterations_to_correct, r.total_policy_evals) == \
        (ref.conflicts, ref.iterations_to_correct, ref.total_policy_evals)


def test_sequential_drop_in_matches_oracle():
    for J, I, T in ((10, 100, 5000), (40, 50, 3000)):
        ons, inst, owner, opol, pol = _dual_case(J, I, T, 8, "product")
        seq, _ = ORC.sequential(ons, opol)
        out = P.sequential_simulate(inst, pol)
        assert out.actions.tolist() == seq.tolist()
        assert out.policy_evals == T


def test_windowed_runs_and_warm_starts_match_oracle():
    ons, inst, owner, opol, pol = _dual_case(10, 50, 3000, 32, "product")
    seq, _ = ORC.sequential(ons, opol)
    draft, _ = ORC.sequential(ons, NS(kind=1, hidden=64, gamma=2.0, horizon=None))
    for ms in (1, 7, 300, 0):
        for init in (None, draft):
            want = ORC.picard(ons, opol, owner, 32, max_steps=ms, record_trace=True, reference=seq,
                              initial_cache=init)
            r = P.picard_simulate(inst, pol, P.PartitionPlan(32, owner),
                                  P.PicardConfig(max_steps=ms, record_trace=True), init, seq)
            assert r.actions.tolist() == seq.tolist()
            assert [x.astuple() for x in r.trace] == [tuple(x) for x in want.trace]
            assert (r.conflicts, r.iterations_to_correct) == (want.conflicts, want.iterations_to_correct)


def test_iteration_cap_raises_with_partial_trace():
    # test_engine.cpp:525-545
    toy = P.Instance(2, 1, 2, [0, 0], [0, 1], [[0.9, 0.1], [0.8, 0.2]], [1, 1], [[1, 1]])
    with pytest.raises(P.IterationLimitError) as e:
        P.picard_simulate(toy, P.GreedyPolicy(), P.PartitionPlan(2, [0, 1]),
                          P.PicardConfig(max_iterations=1, record_trace=True))
    assert e.value.iterations_run == 1 and len(e.value.partial_trace) == 1


def test_plan_and_config_validation():
    # test_engine.cpp:416-453
    toy = P.Instance(2, 1, 2, [0, 0], [0, 1], [[0.9, 0.1], [0.8, 0.2]], [1, 1], [[1, 1]])
    g = P.GreedyPolicy()
    with pytest.raises(P.ContractViolation):
        P.picard_simulate(toy, g, P.PartitionPlan(2, [0]))
    with pytest.raises(P.ContractViolation):
        P.picard_simulate(toy, g, P.PartitionPlan(2, [0, 5]))
    with pytest.raises(P.ContractViolation):
        P.picard_simulate(toy, g, P.PartitionPlan(2, [0, 1]), P.PicardConfig(processes=3))
    with pytest.raises(P.ContractViolation):
        P.picard_simulate(toy, g, P.PartitionPlan(2, [0, 1]), initial_cache=[-1])
    r = P.picard_simulate(toy, g, P.PartitionPlan(3, []) if False else P.PartitionPlan(2, [0, 1]))
    assert r.actions.tolist() == [0, 1]


def test_empty_horizon():
    inst = P.Instance(2, 1, 0, [], [], [[0.5, 0.5]], [1, 1], [[1, 1]])
    r = P.picard_simulate(inst, P.GreedyPolicy(), P.PartitionPlan(3, []))
    assert r.actions.size == 0 and r.iterations_to_converged == 0 and r.total_policy_evals == 0


def test_nonfinite_dual_scores_raise_like_the_reference():
    J = 3
    ons = NS(**ORC.generate_instance_arrays(J, 4, 50, 0.0, 0.8, 3))
    inst = product_instance(ons)
    params = P.MlpParams.seeded_uniform(7, 6, 9)
    params.b3 = params.b3.copy()
    params.b3[1] = np.inf
    pol = P.DualNetworkPolicy(params, nodes=J)
    opol = NS(kind=2, hidden=64, gamma=0.0, horizon=None, w1=params.w1, b1=params.b1, w2=params.w2,
              b2=params.b2, w3=params.w3, b3=params.b3)
    with pytest.raises(OracleError) as oe:
        ORC.sequential(ons, opol)
    with pytest.raises(P.ContractViolation) as ge:
        P.sequential_simulate(inst, pol)
    assert ge.value.time_step == oe.value.time_step
    owner = ORC.uniform_partition(50, 3, 1)
    with pytest.raises(OracleError) as oe2:
        ORC.picard(ons, opol, owner, 3)
    with pytest.raises(P.ContractViolation) as ge2:
        P.picard_simulate(inst, pol, P.PartitionPlan(3, owner))
    assert ge2.value.time_step == oe2.value.time_step


def test_zero_network_equals_greedy():
    # test_policies.cpp:117-132
    ons = NS(**ORC.generate_instance_arrays(5, 12, 800, -0.5, 0.8, 5))
    inst = product_instance(ons)
    a = P.sequential_simulate(inst, P.DualNetworkPolicy.zero(inst)).actions
    b = P.sequential_simulate(inst, P.GreedyPolicy()).actions
    assert a.tolist() == b.tolist()


def test_full_scale_c3_prefix_and_feasibility():
    """C3 shape (J=100, I=1e4, T=1e7 needs minutes of oracle time); at a reduced
    T with the C3 per-product density the GPU trajectory must (a) equal the
    serial oracle on a prefix, (b) be a feasible trajectory, (c) conserve
    units (test_fo_env.cpp:71-106)."""
    J, I, T = 100, 1000, 1_000_000
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    plan = P.make_product_partition(inst, 4096, 1)
    r = P.picard_simulate(inst, pol, plan)
    ons = NS(nodes=J, products=I, horizon=200_000, product=inst.product[:200_000], order_t=None,
             reward_row=inst.reward_row[:200_000], reward_table=inst.reward_table.ravel(),
             capacity=inst.capacity, inventory=inst.inventory.ravel())
    opol = NS(kind=2, hidden=64, gamma=0.0, horizon=T, w1=pol.w1, b1=pol.b1, w2=pol.w2, b2=pol.b2,
              w3=pol.w3, b3=pol.b3)
    seq_prefix, _ = ORC.sequential(ons, opol)
    assert r.actions[:200_000].tolist() == seq_prefix.tolist()
    cap = inst.capacity.astype(np.int64).copy()
    inv = inst.inventory.astype(np.int64).copy()
    a = r.actions
    ok = a >= 0
    np.subtract.at(cap, a[ok], 1)
    np.subtract.at(inv, (inst.product[ok], a[ok]), 1)
    assert cap.min() >= 0 and inv.min() >= 0
    assert int(ok.sum()) == int(inst.capacity.sum() - cap.sum())


def test_c3_chunk_and_product_plans_agree():
    """The bench workload (C3: J=100, I=1e4, T=1e7): the product-chunk plan and
    the reference's product plan (both on the tensor-core engine, whole-horizon
    window) reach the same trajectory in the same 66 iterations; the
    reference pin of that trajectory (all 1e7 actions, reward, final state,
    verify mode, FP64 engine) is tests/test_gpu_fullscale.py."""
    J, I, T = 100, 10_000, 10_000_000
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    cfg = P.PicardConfig(max_steps=300 * 65536)
    chunk = P.picard_simulate(inst, pol, P.make_product_chunk_partition(inst, 65536, 1), cfg)
    prod = P.picard_simulate(inst, pol, P.make_product_partition(inst, 65536, 1), cfg)
    assert np.array_equal(chunk.actions, prod.actions)
    assert chunk.iterations_to_converged == prod.iterations_to_converged == 66
    assert chunk.timing["tc_used"] == 1 and prod.timing["tc_used"] == 1


@pytest.mark.parametrize("J,I,T,M", [(10, 300, 20000, 512), (30, 200, 12000, 256), (100, 40, 4000, 64),
                                     (100, 300, 30000, 512), (1, 10, 10000, 16), (3, 7, 900, 5)])
def test_tensor_core_sweep_matches_oracle(J, I, T, M):
    """The tcgen05 fp16x3 policy path with the FP64 margin recheck must give the
    reference's exact trajectory and per-iteration counters; in verify mode no
    unflagged row may disagree with the exact FP64 decision."""
    ons, inst, owner, opol, pol = _dual_case(J, I, T, M, "product")
    seq, _ = ORC.sequential(ons, opol)
    want = ORC.picard(ons, opol, owner, M, record_trace=True, reference=seq)
    for verify in (False, True):
        r = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner),
                              P.PicardConfig(record_trace=True, engine="product", tc_verify=verify),
                              reference_actions=seq)
        assert r.timing["tc_used"] == 1
        assert r.timing["tc_rows"] > 0
        assert r.timing["tc_unflagged_bad"] == 0
        assert r.actions.tolist() == seq.tolist()
        assert r.iterations_to_converged == want.iterations_to_converged
        assert r.iterations_to_correct == want.iterations_to_correct
        assert r.conflicts == want.conflicts
        assert r.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent
        assert r.total_policy_evals == want.total_policy_evals
        assert [x.astuple() for x in r.trace] == [tuple(x) for x in want.trace]


def test_tensor_core_and_fp64_sweeps_agree_with_warm_start_and_windows():
    ons, inst, owner, opol, pol = _dual_case(10, 80, 8000, 128, "product")
    draft, _ = ORC.sequential(ons, NS(kind=1, hidden=64, gamma=2.0, horizon=None))
    for ms in (0, 250):
        a = P.picard_simulate(inst, pol, P.PartitionPlan(128, owner),
                              P.PicardConfig(max_steps=ms, record_trace=True, engine="product"), draft)
        b = P.picard_simulate(inst, pol, P.PartitionPlan(128, owner),
                              P.PicardConfig(max_steps=ms, record_trace=True, engine="product_fp64"), draft)
        assert a.timing["tc_used"] == 1 and b.timing["tc_used"] == 0
        assert a.actions.tolist() == b.actions.tolist()
        assert [x.astuple() for x in a.trace] == [x.astuple() for x in b.trace]


@pytest.mark.parametrize("J,I,T,M,kind", [(10, 100, 6000, 64, 2), (30, 300, 8000, 200, 2), (12, 50, 5000, 40, 0),
                                           (12, 50, 5000, 40, 1), (6, 20, 4000, 7, 2)])
def test_general_engine_uniform_plans_match_replay(J, I, T, M, kind):
    """Uniform plans (not run partitions): the general closed form reproduces
    the exact replay sweep iteration by iteration and converges to the serial
    trajectory."""
    ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, 3, geometry=0))
    inst = product_instance(ons)
    owner = ORC.uniform_partition(T, M, 2)
    spec = dict(kind=kind, gamma=1.3, seed=5)
    opol, pol = oracle_policy(spec, ons, ORC), product_policy(spec, inst)
    seq, _ = ORC.sequential(ons, opol)
    rs = {e: P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(record_trace=True, engine=e),
                               reference_actions=seq) for e in ("replay", "general")}
    for r in rs.values():
        assert r.actions.tolist() == seq.tolist()
    assert [x.astuple() for x in rs["general"].trace] == [x.astuple() for x in rs["replay"].trace]
    assert (rs["general"].conflicts, rs["general"].total_policy_evals) == (rs["replay"].conflicts,
                                                                         rs["replay"].total_policy_evals)
    assert rs["general"].timing["engine_used"] == 4


@pytest.mark.parametrize("scale,shrink,tc", [(2.0, 1, 1), (1.0, 4, 1), (3.0, 2, 1), (8.0, 1, 0), (float("nan"), 1, 0)])
def test_tensor_core_guard_scales_with_policy(scale, shrink, tc):
    """Policies with larger weights / features than the reference's seeded
    ones: the tensor-core guard grows with their error propagation (verify
    mode: no unflagged disagreement), and policies whose error bound is too
    large, or whose weights are not finite, keep the exact FP64 path."""
    ons, inst, owner, _, _ = _dual_case(30, 200, 12000, 256, "product")
    p = P.MlpParams.seeded_uniform(61, 60, 5)
    for a in (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3):
        a *= 1.0 if scale != scale else scale
    if scale != scale:
        p.w1[3 * 61 + 7] = float("nan")
    cap0 = np.maximum(np.asarray(inst.capacity) // shrink, 1)
    inv0 = np.asarray(inst.inventory) // shrink
    pol = P.DualNetworkPolicy(p, cap0, inv0, inst.horizon, 30)
    plan = P.PartitionPlan(256, owner)
    runs = {}
    for engine, verify in (("product", False), ("product", True), ("product_fp64", False)):
        try:
            r = P.picard_simulate(inst, pol, plan, P.PicardConfig(record_trace=True, engine=engine, tc_verify=verify))
            runs[(engine, verify)] = (r.actions.tolist(), [x.astuple() for x in r.trace], r.timing)
        except P.ContractViolation as e:
            runs[(engine, verify)] = ("ContractViolation", e.time_step, None)
    base = runs[("product_fp64", False)]
    for key in (("product", False), ("product", True)):
        assert runs[key][:2] == base[:2], key
        if runs[key][2] is not None:
            assert runs[key][2]["tc_used"] == tc
            assert runs[key][2]["tc_unflagged_bad"] == 0
    if tc:  # rows within the guard: re-evaluated in the sweep or speculated and verified after it
        t = runs[("product", False)][2]
        assert t["tc_flagged"] + t["tc_speculated"] > 0


def test_cpp_dropin_matches_reference_engine():
    """The reference's own engine scenarios through include/picard_b200.hpp,
    checked against the UNMODIFIED reference CPU engine (tests/cpp)."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(__file__), "cpp", "_build", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp/_build/dropin_test not built (needs the reference tree)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


def test_single_rank_nccl_path_matches():
    """The multi-GPU exchange (pack -> ncclAllGather -> unpack, scalar
    all-reduces) exercised with a one-rank communicator: identical results."""
    ons, inst, owner, opol, pol = _dual_case(30, 200, 12000, 256, "product")
    seq, _ = ORC.sequential(ons, opol)
    want = P.picard_simulate(inst, pol, P.PartitionPlan(256, owner), P.PicardConfig(record_trace=True),
                             reference_actions=seq)
    uid = P.nccl_unique_id()
    for engine in ("auto", "product_fp64", "replay", "general"):
        with P.Simulator(inst, pol) as sim:
            sim.set_plan(P.PartitionPlan(256, owner))
            sim.attach_comm(uid if engine == "auto" else P.nccl_unique_id(), 0, 1)
            r = sim.simulate(P.PicardConfig(record_trace=True, engine=engine), reference_actions=seq)
        assert r.actions.tolist() == seq.tolist()
        assert [x.astuple() for x in r.trace] == [x.astuple() for x in want.trace]
        assert (r.conflicts, r.iterations_to_correct) == (want.conflicts, want.iterations_to_correct)


@pytest.mark.parametrize("J,I,T,M,scale,shrink", [(10, 300, 20000, 512, 1.0, 1), (30, 200, 12000, 256, 1.0, 1),
                                                   (30, 200, 12000, 256, 2.0, 1), (30, 200, 12000, 256, 1.0, 4),
                                                   (30, 200, 12000, 256, 3.0, 2), (100, 300, 30000, 512, 1.0, 1)])
def test_derived_guard_bounds_the_observed_score_error(J, I, T, M, scale, shrink):
    """The tensor-core guard is derived (tc_error_bound: split / rounding
    errors, the measured tcgen05 accumulation and tanh_mufu errors, weight-wise
    propagation), not calibrated: in verify mode every row is re-evaluated in
    FP64 and the largest observed |score_tc - score_exact| must stay below the
    a-priori bound B; the sweep's margin guard bounds score differences."""
    ons, inst, owner, _, _ = _dual_case(J, I, T, M, "product")
    p = P.MlpParams.seeded_uniform(2 * J + 1, 2 * J, 5)
    for a in (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3):
        a *= scale
    cap0 = np.maximum(np.asarray(inst.capacity) // shrink, 1)
    inv0 = np.asarray(inst.inventory) // shrink
    pol = P.DualNetworkPolicy(p, cap0, inv0, inst.horizon, J)
    B, guard = P.tc_error_bound(inst, pol)
    # the margin guard bounds the error of a DIFFERENCE of two scores of one
    # row (shared hidden-layer error): between B and 2B (times 1 + 2^-10)
    assert B > 0 and B < guard <= 2 * B * (1 + 2 ** -10)
    fp64 = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(engine="product_fp64"))
    r = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(engine="product", tc_verify=True))
    t = r.timing
    assert t["tc_used"] == 1 and t["tc_rows"] > 0
    assert t["tc_score_bound"] == B and t["tc_guard"] == guard
    assert t["tc_unflagged_bad"] == 0
    assert 0 < t["tc_max_score_err"] <= B, (t["tc_max_score_err"], B)
    assert r.actions.tolist() == fp64.actions.tolist()
    print(f"J={J} scale={scale} shrink={shrink}: B={B:.3e} observed max {t['tc_max_score_err']:.3e} "
          f"(B / observed = {B / t['tc_max_score_err']:.0f})")


@pytest.mark.parametrize("shape", ["positive_w1", "positive_all", "heavy_tail", "large_bias", "sparse"])
def test_derived_guard_holds_for_adversarial_weights(shape):
    """Weight structures built to make the tensor-core errors large and
    aligned (all-positive layers: every fp32 truncation goes the same way;
    heavy tails; large biases; sparse rows): the observed max |score error|
    in verify mode stays below the a-priori bound B, no accepted decision
    differs from the FP64 engine, and policies whose guard would be too
    large keep the FP64 path."""
    J, I, T, M = 30, 200, 12000, 256
    ons, inst, owner, _, _ = _dual_case(J, I, T, M, "product")
    rng = np.random.default_rng({"positive_w1": 1, "positive_all": 2, "heavy_tail": 3, "large_bias": 4,
                                 "sparse": 5}[shape])
    p = P.MlpParams.seeded_uniform(2 * J + 1, 2 * J, 5)
    if shape == "positive_w1":
        p.w1 = np.abs(p.w1)
    elif shape == "positive_all":
        p.w1, p.w2, p.w3 = np.abs(p.w1), np.abs(p.w2), np.abs(p.w3)
    elif shape == "heavy_tail":
        for name in ("w1", "w2", "w3"):
            a = getattr(p, name)
            setattr(p, name, a * np.minimum(rng.pareto(1.5, a.shape) + 1.0, 20.0) / 3.0)
    elif shape == "large_bias":
        p.b1 = p.b1 * 30.0
        p.b2 = p.b2 * 30.0
        p.b3 = p.b3 * 10.0
    else:
        for name in ("w1", "w2", "w3"):
            a = getattr(p, name)
            setattr(p, name, np.where(rng.random(a.shape) < 0.8, 0.0, a * 3.0))
    pol = P.DualNetworkPolicy(p, None, None, inst.horizon, J)
    B, guard = P.tc_error_bound(inst, pol)
    fp64 = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(engine="product_fp64"))
    r = P.picard_simulate(inst, pol, P.PartitionPlan(M, owner), P.PicardConfig(engine="product", tc_verify=True))
    t = r.timing
    assert r.actions.tolist() == fp64.actions.tolist()
    assert t["tc_unflagged_bad"] == 0
    if guard > 0:
        assert t["tc_used"] == 1
        assert t["tc_max_score_err"] <= B, (t["tc_max_score_err"], B)
        print(f"{shape}: B={B:.3e} guard={guard:.3e} observed={t['tc_max_score_err']:.3e} "
              f"flagged={t['tc_flagged'] / max(t['tc_rows'], 1):.2%}")
    else:
        assert t["tc_used"] == 0
        print(f"{shape}: B={B:.3e}: FP64 path")
