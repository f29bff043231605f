"""Time Warp safe-window baseline (timewarp::time_warp_simulate,
fo/timewarp.hpp:56-181) on the device against the UNMODIFIED reference
(oracle/_ref): actions, sync rounds, rollbacks, evaluation counters and trace
rows must be identical, for both window rules and all policy kinds,
including the reference test suite's cases (test_timewarp.cpp)."""
from types import SimpleNamespace as NS

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import ORC, REF
from tests.helpers import oracle_policy, product_instance, product_policy

pytestmark = pytest.mark.gpu


def _check(ons, spec, processes, seed, rule):
    inst = product_instance(ons)
    opol = oracle_policy(spec, ons, ORC)
    pol = product_policy(spec, inst)
    want_a, want_c, want_tr = REF.time_warp(ons, opol, processes, seed, rule=rule)
    got = P.time_warp_simulate(inst, pol, processes, seed, record_trace=True,
                               rule="min_stocked_capacity" if rule else "min_capacity")
    assert got.actions.tolist() == want_a.tolist()
    assert [got.sync_rounds, got.rollbacks, got.policy_eval_count_sequential_equivalent,
            got.total_policy_evals] == want_c.tolist()
    assert [r.astuple() for r in got.trace] == [tuple(int(x) for x in row) for row in want_tr]
    return got


@pytest.mark.parametrize("seed", [60, 61, 62, 63, 55, 72])
@pytest.mark.parametrize("rule", [0, 1])
def test_small_random_instances_match_reference(seed, rule):
    J, I, T, beta, cov, s = ORC.small_random_params(seed)
    ons = NS(**ORC.generate_instance_arrays(J, I, T, beta, cov, s))
    for spec in (dict(kind=0, gamma=0.0, seed=None), dict(kind=1, gamma=5.0, seed=None),
                 dict(kind=2, gamma=0.0, seed=seed)):
        _check(ons, spec, 4, seed, rule)


@pytest.mark.parametrize("J,I,T,M,kind", [(5, 1500, 4000, 64, 0), (10, 300, 20000, 128, 2), (30, 200, 12000, 256, 2),
                                          (100, 40, 4000, 16, 2), (10, 100, 8000, 32, 1)])
def test_generated_instances_match_reference(J, I, T, M, kind):
    ons = NS(**ORC.generate_instance_arrays(J, I, T, 0.0, 0.8, 9, geometry=0 if J <= 30 else 1))
    for rule in (0, 1):
        got = _check(ons, dict(kind=kind, gamma=1.5, seed=5), M, 9, rule)
        assert got.rollbacks == 0


def test_no_capacity_network_completes():
    ons = NS(nodes=2, products=2, horizon=6, product=np.array([0, 1, 0, 1, 0, 1], np.int32), order_t=None,
             reward_row=np.zeros(6, np.int32), reward_table=np.array([0.5, 0.5]), capacity=np.zeros(2, np.int32),
             inventory=np.full(4, 4, np.int32))
    for rule in (0, 1):
        got = _check(ons, dict(kind=0, gamma=0.0, seed=None), 2, 1, rule)
        assert (got.actions == -1).all()
