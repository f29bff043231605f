"""Timing of the general closed-form engine on C3-shaped plans (not a test):
the product-chunk plan (long same-product runs), the uniform time partition,
and a product partition with a fraction of slots reassigned at random (a
plan that is neither). One JSON line per plan.

  python tools/general_probe.py [T]
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

J, I, M = 100, 10_000, 65536
T = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
rng = np.random.default_rng(3)
mixed = P.make_product_partition(inst, 4096, 1).owner.copy()
flip = rng.random(T) < 0.01
mixed[flip] = rng.integers(0, 4096, int(flip.sum()))
plans = {"chunk": P.make_product_chunk_partition(inst, M, 1), "uniform": P.make_uniform_time_partition(T, M, 1),
         "product4096+1%": P.PartitionPlan(4096, mixed)}
seq = None
for name, plan in plans.items():
    with P.Simulator(inst, pol) as sim:
        sim.set_plan(plan)
        r = sim.simulate_resident(P.PicardConfig(max_steps=300 * plan.processes, engine="general"))
        acts = sim.download_actions()
    seq = acts if seq is None else seq
    tm = r.timing
    print(json.dumps(dict(plan=name, T=T, M=plan.processes, iterations=r.iterations_to_converged, ms=tm["total_ms"],
                          sweep_ms=tm["sweep_ms"], prep_ms=tm["prep_ms"], evals=r.total_policy_evals,
                          steps_per_s=T / (tm["total_ms"] / 1000.0), same_trajectory=bool((acts == seq).all()))),
          flush=True)
