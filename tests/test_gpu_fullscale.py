"""Full-size parity pins against the UNMODIFIED reference (oracle/_ref).

* C3 (BASELINE configs[2], the bench workload: J=100, I=1e4, T=1e7, 65536
  processes): the instance and policy built by the product equal the
  reference generator's; the whole 1e7-step trajectory equals the
  reference's sequential_simulate (engine.hpp:237-267) action for action, on
  the tensor-core engine at the bench's window and at the CLI-default window
  (equal-count chunks and the bench's window-aware chunks),
  and on the FP64 SIMT engine; fo_total_reward agrees (rel. 1e-4 is the
  north-star bar; the difference is printed); the final FoState (the device
  checkpoint after convergence) equals the reference's state after the
  serial run; in verify mode no tensor-core decision that escaped the exact
  recheck disagrees with FP64.
* C2 (configs[1]: J=10, I=1e3, T=1e6, M=4096): picard_simulate's counters
  and trace (iterations to converged / correct, conflicts, evaluation
  counters, every trace row) equal the reference's picard_simulate
  (engine.hpp:458-590, threads = every host core) on the reference's
  product partition, the product-chunk plan and the window-aware chunk plan.

The reference serial run at C3 takes ~2-3 min on one host core.
"""
import os
from types import SimpleNamespace as NS

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import REF

pytestmark = [pytest.mark.gpu, pytest.mark.slow,
              pytest.mark.skipif(REF is None, reason="oracle/_ref (the compiled reference) is not built")]

C3 = (100, 10_000, 10_000_000, 65536)
C3_WINDOW = 350_000  # bench.py WINDOWS["c3"]


def _opol(pol, T):
    return NS(kind=2, hidden=64, gamma=0.0, horizon=T, w1=pol.w1, b1=pol.b1, w2=pol.w2, b2=pol.b2,
              w3=pol.w3, b3=pol.b3)


@pytest.fixture(scope="module")
def c3():
    J, I, T, M = C3
    ref = NS(**REF.generate_instance_arrays(J, I, T, 0.0, 0.8, 7, geometry=1))
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    for k in ("product", "reward_row", "capacity"):
        assert np.array_equal(getattr(inst, k), getattr(ref, k)), k
    assert np.array_equal(inst.inventory.ravel(), ref.inventory)
    assert np.array_equal(inst.reward_table.ravel(), ref.reward_table)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    w = REF.seeded_mlp(2 * J + 1, 2 * J, 5)
    for a, b in zip((pol.w1, pol.b1, pol.w2, pol.b2, pol.w3, pol.b3), w):
        assert np.array_equal(a, b)
    sess = REF.session(ref, _opol(pol, T))
    seq, sec = sess.run(T)
    _, _, cap, inv = sess.state()
    reward = sess.total_reward(seq)
    sess.close()
    print(f"\nreference sequential_simulate over the full C3 horizon: {sec:.1f} s")
    plan = P.make_product_chunk_partition(inst, M, 1)
    wplan = P.make_product_window_partition(inst, M, C3_WINDOW, 1)  # the bench's plan
    return NS(ref=ref, inst=inst, pol=pol, seq=seq, cap=cap, inv=inv, reward=reward, plan=plan, wplan=wplan)


@pytest.mark.parametrize("window,engine,kernel,plan", [(C3_WINDOW, "auto", "fused", "window"),
                                                       (C3_WINDOW, "auto", "fused", "chunk"),
                                                       (C3_WINDOW, "auto", "incremental", "chunk"),
                                                       (500_000, "auto", "fused", "chunk"),
                                                       (300 * 65536, "auto", "fused", "chunk"),
                                                       (300 * 65536, "auto", "fused", "window"),
                                                       (300 * 65536, "auto", "incremental", "chunk"),
                                                       (300 * 65536, "product_fp64", "auto", "chunk")])
def test_c3_full_trajectory_equals_reference_serial(c3, window, engine, kernel, plan):
    with P.Simulator(c3.inst, c3.pol) as sim:
        sim.set_plan(c3.wplan if plan == "window" else c3.plan)
        r = sim.simulate(P.PicardConfig(max_steps=window, engine=engine, tc_kernel=kernel))
        cap, inv = sim.checkpoint_state()
    assert r.timing["tc_used"] == (1 if engine == "auto" else 0)
    first = np.flatnonzero(r.actions != c3.seq)
    assert first.size == 0, f"first mismatch at t={first[0]}"
    assert np.array_equal(cap, c3.cap)
    assert np.array_equal(inv.ravel(), c3.inv)
    got = P.fo_total_reward(c3.inst, r.actions)
    rel = abs(got - c3.reward) / max(1.0, abs(c3.reward))
    print(f"\nC3 window={window} engine={engine} kernel={kernel}: {r.iterations_to_converged} iterations, "
          f"total reward {got!r} vs reference {c3.reward!r} (rel. diff {rel:.3e})")
    assert rel <= 1e-4


@pytest.mark.parametrize("window,kernel,plan", [(C3_WINDOW, "fused", "window"), (C3_WINDOW, "fused", "chunk"),
                                                (C3_WINDOW, "incremental", "chunk"), (300 * 65536, "fused", "chunk")])
def test_c3_verify_mode_every_row_rechecked(c3, window, kernel, plan):
    """tc_verify: every tensor-core row is also evaluated in exact FP64; no row
    outside the guard may disagree (tc_unflagged_bad == 0) and the trajectory
    is the reference's."""
    with P.Simulator(c3.inst, c3.pol) as sim:
        sim.set_plan(c3.wplan if plan == "window" else c3.plan)
        r = sim.simulate(P.PicardConfig(max_steps=window, tc_verify=True, tc_kernel=kernel))
    t = r.timing
    assert t["tc_used"] == 1 and t["tc_rows"] > 3e7
    assert t["tc_unflagged_bad"] == 0
    assert np.array_equal(r.actions, c3.seq)
    print(f"\nverify window={window} kernel={kernel}: {t['tc_rows']} rows, {t['tc_flagged']} flagged, "
          f"{t['tc_disagree']} flagged rows where fp16x3 was wrong, 0 unflagged wrong")


@pytest.fixture(scope="module")
def c2():
    J, I, T, M = 10, 1000, 1_000_000, 4096
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    ref = NS(**REF.generate_instance_arrays(J, I, T, 0.0, 0.8, 7))
    assert np.array_equal(inst.product, ref.product) and np.array_equal(inst.inventory.ravel(), ref.inventory)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    seq, _ = REF.sequential(ref, _opol(pol, T))
    return NS(inst=inst, ref=ref, pol=pol, seq=seq, M=M, T=T)


@pytest.mark.parametrize("part,window", [("product", 0), ("chunk", 0), ("chunk", 100_000), ("window", 100_000)])
def test_c2_counters_and_trace_equal_reference_picard(c2, part, window):
    if part == "product":
        plan = P.make_product_partition(c2.inst, c2.M, 1)
        assert np.array_equal(plan.owner, REF.product_partition(c2.ref, c2.M, 1))
    elif part == "window":
        plan = P.make_product_window_partition(c2.inst, c2.M, window, 1)
    else:
        plan = P.make_product_chunk_partition(c2.inst, c2.M, 1)
    ms = window or 300 * c2.M
    want = REF.picard(c2.ref, _opol(c2.pol, c2.T), plan.owner, c2.M, max_steps=ms, record_trace=True,
                      threads=os.cpu_count() or 1, reference=c2.seq)
    got = P.picard_simulate(c2.inst, c2.pol, plan, P.PicardConfig(max_steps=ms, record_trace=True),
                            reference_actions=c2.seq)
    assert np.array_equal(want.actions, c2.seq)
    assert np.array_equal(got.actions, c2.seq)
    assert got.iterations_to_converged == want.iterations_to_converged
    assert got.iterations_to_correct == want.iterations_to_correct
    assert got.conflicts == want.conflicts
    assert got.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent
    assert got.total_policy_evals == want.total_policy_evals
    assert [x.astuple() for x in got.trace] == [tuple(x) for x in want.trace]
    print(f"\nC2 {part} window={ms}: {got.iterations_to_converged} iterations "
          f"({got.iterations_to_correct} to correct), {got.total_policy_evals} evaluations")
