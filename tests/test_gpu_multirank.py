"""The multi-GPU protocol executed for real on one GPU.

N handles on the same device, each driven by its own host thread and
attached to an in-process loopback group (pcd_attach_loopback), run exactly
the code a torchrun job runs per rank: LPT process shards (rebuild_shards),
the per-rank process masks in every sweep, pack -> all-gather of each rank's
owned window slots -> unpack, and the integer all-reduces of the convergence
scalars (engine.cu exchange()). Only the transport differs from NCCL (device
copies through a staging buffer). Every rank must return the single-rank
result bit for bit: actions, counters and every trace row."""
import threading
from types import SimpleNamespace as NS

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import ORC
from tests.helpers import product_instance

pytestmark = pytest.mark.gpu


def _case(J, I, T, seed=7):
    ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, seed))
    inst = product_instance(ons)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    opol = NS(kind=2, hidden=64, gamma=0.0, horizon=None, w1=pol.w1, b1=pol.b1, w2=pol.w2, b2=pol.b2,
              w3=pol.w3, b3=pol.b3)
    seq, _ = ORC.sequential(ons, opol)
    return inst, pol, seq


def _run_ranks(inst, pol, plan, cfg, seq, nranks):
    group = P.LoopbackGroup(nranks)
    sims = [P.Simulator(inst, pol) for _ in range(nranks)]
    for r, sim in enumerate(sims):
        sim.set_plan(plan)
        sim.attach_loopback(group, r)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            out[r] = sims[r].simulate(cfg, reference_actions=seq)
        except Exception as e:  # surfaced below
            errs.append(e)

    threads = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
    for sim in sims:
        sim.close()
    group.close()
    if errs:
        raise errs[0]
    return out


def _same(a, b):
    assert np.array_equal(a.actions, b.actions)
    assert (a.iterations_to_converged, a.iterations_to_correct, a.conflicts,
            a.policy_eval_count_sequential_equivalent, a.total_policy_evals) == \
        (b.iterations_to_converged, b.iterations_to_correct, b.conflicts,
         b.policy_eval_count_sequential_equivalent, b.total_policy_evals)
    assert [x.astuple() for x in a.trace] == [x.astuple() for x in b.trace]


@pytest.mark.parametrize("nranks", [2, 4, 8])
@pytest.mark.parametrize("engine,part,window", [("auto", "product", 0), ("auto", "product", 2500),
                                                ("product_fp64", "product", 0), ("general", "product", 3000),
                                                ("replay", "product", 0), ("auto", "uniform", 0),
                                                ("auto", "chunk", 1500), ("auto", "window", 1500)])
def test_loopback_ranks_equal_single_rank(nranks, engine, part, window):
    inst, pol, seq = _case(30, 200, 12000)
    M = 256
    if part == "product":
        plan = P.make_product_partition(inst, M, 1)
    elif part == "chunk":
        plan = P.make_product_chunk_partition(inst, M, 1)
    elif part == "window":
        plan = P.make_product_window_partition(inst, M, window, 1)
    else:
        plan = P.make_uniform_time_partition(inst.horizon, 64, 1)
    cfg = P.PicardConfig(max_steps=window, record_trace=True, engine=engine)
    want = P.picard_simulate(inst, pol, plan, cfg, reference_actions=seq)
    assert np.array_equal(want.actions, seq)
    for r in _run_ranks(inst, pol, plan, cfg, seq, nranks):
        _same(r, want)


@pytest.mark.parametrize("nranks", [2, 8])
def test_loopback_ranks_c2_shape(nranks):
    """C2 (J=10, I=1e3, T=1e6, M=4096 product-chunk plan) on the tensor-core
    engine with a 100k-slot window: the shards carry real work per rank."""
    inst = P.generate_instance(10, 1000, 1_000_000, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    plan = P.make_product_chunk_partition(inst, 4096, 1)
    cfg = P.PicardConfig(max_steps=100_000, record_trace=True)
    want = P.picard_simulate(inst, pol, plan, cfg)
    shards = P.shard_processes(plan, nranks)
    loads = np.bincount(shards[plan.owner], minlength=nranks)
    assert loads.min() > 0 and loads.max() <= 1.01 * loads.mean()
    for r in _run_ranks(inst, pol, plan, cfg, None, nranks):
        _same(r, want)
