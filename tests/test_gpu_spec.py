"""Speculative tensor-core decisions (tc_spec.cu): rows whose margins lie
between 1/256 of the derived guards and the guards take the tensor-core
decision at once and are verified against the reference policy after the
sweep; a wrong one re-runs the iteration without speculation. Results must be
identical to the non-speculative sweep (PCD_DEBUG_NO_SPEC) -- actions,
counters, every trace row -- and to the oracle, also when every speculated
decision is forced to count as wrong (PCD_DEBUG_SPEC_RERUN: every iteration
with a speculated row is re-run from its backups), and when every 4th
speculated decision is published wrong on purpose (PCD_DEBUG_SPEC_FLIP: the
verification must detect each such iteration and re-run it)."""
from types import SimpleNamespace as NS

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import ORC
from tests.helpers import product_instance

pytestmark = pytest.mark.gpu

NO_SPEC, SPEC_RERUN, SPEC_FLIP = 8, 16, 32


def _case(J, I, T, seed=7, scale=1.0):
    ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, seed, geometry=0 if J <= 30 else 1))
    inst = product_instance(ons)
    p = P.MlpParams.seeded_uniform(2 * J + 1, 2 * J, 5)
    for a in (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3):
        a *= scale
    pol = P.DualNetworkPolicy(p, None, None, inst.horizon, J)
    opol = NS(kind=2, hidden=64, gamma=0.0, horizon=None, w1=pol.w1, b1=pol.b1, w2=pol.w2, b2=pol.b2,
              w3=pol.w3, b3=pol.b3)
    return ons, inst, pol, opol


def _run(inst, pol, plan, cfg, flags, seq=None):
    with P.Simulator(inst, pol) as sim:
        sim.set_plan(plan)
        P._capi.LIB.pcd_set_debug(sim._h, flags)
        return sim.simulate(cfg, reference_actions=seq)


@pytest.mark.parametrize("J,I,T,M,part,window,scale", [(30, 200, 12000, 256, "product", 0, 1.0),
                                                        (30, 200, 12000, 256, "chunk", 2000, 2.0),
                                                        (100, 300, 30000, 512, "chunk", 0, 1.0),
                                                        (100, 300, 30000, 512, "chunk", 5000, 1.0),
                                                        (10, 1000, 200000, 2048, "chunk", 20000, 1.0),
                                                        (30, 200, 12000, 512, "window", 2000, 1.0),
                                                        (100, 300, 30000, 1024, "window", 5000, 1.0)])
def test_speculation_equals_the_non_speculative_sweep(J, I, T, M, part, window, scale):
    ons, inst, pol, opol = _case(J, I, T, scale=scale)
    plan = (P.make_product_chunk_partition(inst, M, 1) if part == "chunk"
            else P.make_product_window_partition(inst, M, window, 1) if part == "window"
            else P.make_product_partition(inst, M, 1))
    seq, _ = ORC.sequential(ons, opol)
    cfg = P.PicardConfig(max_steps=window, record_trace=True)
    runs = {f: _run(inst, pol, plan, cfg, f, seq) for f in (0, NO_SPEC, SPEC_RERUN, SPEC_FLIP)}
    base = runs[NO_SPEC]
    assert base.actions.tolist() == seq.tolist()
    assert base.timing["tc_speculated"] == 0
    for f in (0, SPEC_RERUN, SPEC_FLIP):
        r = runs[f]
        assert r.timing["tc_used"] == 1
        assert r.actions.tolist() == seq.tolist()
        assert (r.iterations_to_converged, r.iterations_to_correct, r.conflicts,
                r.policy_eval_count_sequential_equivalent, r.total_policy_evals) == \
            (base.iterations_to_converged, base.iterations_to_correct, base.conflicts,
             base.policy_eval_count_sequential_equivalent, base.total_policy_evals)
        assert [x.astuple() for x in r.trace] == [x.astuple() for x in base.trace]
    spec, rerun = runs[0].timing, runs[SPEC_RERUN].timing
    assert spec["tc_speculated"] > 0
    assert spec["tc_spec_reruns"] == 0  # (no wrong speculated decision in these cases)
    assert rerun["tc_spec_reruns"] > 0
    assert runs[SPEC_FLIP].timing["tc_spec_reruns"] > 0  # the planted wrong decisions were caught
