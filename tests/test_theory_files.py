"""Depletion profile on the device (theory::compute_depletion) against the
unmodified reference, the iteration bound of the reference's theory tests
(test_theory.cpp:208-226), and the binary SoA instance files."""
from types import SimpleNamespace as NS

import numpy as np
import pytest

import paper_2406_01939_b200 as P
from oracle.oracle import ORC, REF
from tests.helpers import oracle_policy, product_instance


def test_binary_instance_round_trip(tmp_path):
    inst = P.generate_instance(10, 50, 3000, -0.4, 0.8, 3)
    f = tmp_path / "a.pcd"
    P.save_instance_binary(inst, f)
    back = P.load_instance_binary(f)
    assert (back.nodes, back.products, back.horizon) == (inst.nodes, inst.products, inst.horizon)
    for name in ("product", "reward_row", "capacity", "inventory"):
        assert np.array_equal(np.asarray(getattr(back, name)).ravel(), np.asarray(getattr(inst, name)).ravel())
    assert np.array_equal(np.asarray(back.reward_table).ravel(), np.asarray(inst.reward_table).ravel())
    # with explicit order times
    inst2 = P.Instance(2, 2, 4, [0, 1, 0, 1], [0, 1, 0, 1], [[1.0, 0.5], [0.25, 2.0]], [3, 3], [[2, 2], [2, 2]],
                       [5, 6, 7, 8])
    P.save_instance_binary(inst2, tmp_path / "b.pcd")
    back2 = P.load_instance_binary(tmp_path / "b.pcd")
    assert np.asarray(back2.order_t).tolist() == [5, 6, 7, 8]
    with pytest.raises(P.InvalidArgument):
        P.load_instance_binary(tmp_path / "missing.pcd")
    (tmp_path / "bad.pcd").write_bytes(b"not an instance file at all, definitely not")
    with pytest.raises(P.InvalidArgument):
        P.load_instance_binary(tmp_path / "bad.pcd")


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(90, 100))
def test_depletion_profile_and_iteration_bound(seed):
    J, I, T, beta, cov, s = ORC.small_random_params(seed)
    ons = NS(**ORC.generate_instance_arrays(J, I, T, beta, cov, s))
    inst = product_instance(ons)
    opol = oracle_policy(dict(kind=0, gamma=0.0, seed=None), ons, ORC)
    seq, _ = ORC.sequential(ons, opol)
    prof = P.depletion_profile(inst, seq)
    assert prof.first_depleted_at.tolist() == REF.depletion(ons, seq).tolist()
    # greedy product-partition runs stay within |Q_T| + 1 (test_theory.cpp:208-226)
    owner = ORC.product_partition(ons, 4, seed)
    r = P.picard_simulate(inst, P.GreedyPolicy(), P.PartitionPlan(4, owner), reference_actions=seq)
    bound, ok = P.check_iteration_bound(r.iterations_to_correct, prof)
    assert ok and bound == prof.depleted_count() + 1


@pytest.mark.gpu
def test_depletion_profile_large_and_edge_cases():
    inst = P.generate_instance(30, 2000, 200_000, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    r = P.picard_simulate(inst, pol, P.make_product_chunk_partition(inst, 4096))
    ons = NS(nodes=inst.nodes, products=inst.products, horizon=inst.horizon, product=inst.product, order_t=None,
             reward_row=inst.reward_row, reward_table=np.asarray(inst.reward_table).ravel(),
             capacity=inst.capacity, inventory=np.asarray(inst.inventory).ravel())
    assert P.depletion_profile(inst, r.actions).first_depleted_at.tolist() == REF.depletion(ons, r.actions).tolist()
    # zero-capacity node depletes at 0; all-decline trajectory never depletes the others
    toy = P.Instance(2, 1, 3, [0, 0, 0], [0, 0, 0], [[1.0, 1.0]], [0, 5], [[3, 3]])
    prof = P.depletion_profile(toy, [-1, -1, -1])
    assert prof.first_depleted_at.tolist() == [0, 3] and prof.iteration_bound() == 2
