"""C3 with debug flag sets (not a test): iterations, speculation re-runs,
speculated rows, evaluations, and whether the actions equal the first run's.
  python tools/spec_ab.py 8 0 16     # no speculation, default, forced re-runs
"""
import sys; sys.path.insert(0,'.')
import numpy as np, paper_2406_01939_b200 as P
inst = P.generate_instance(100, 10000, 10_000_000, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, 65536, 1)
res = {}
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for f in [int(x) for x in sys.argv[1:]] or (8, 0, 16):
        P._capi.LIB.pcd_set_debug(sim._h, f)
        r = sim.simulate(P.PicardConfig(max_steps=300000))
        a = np.asarray(sim.download_actions()).copy()
        res[f] = a
        print(f, r.iterations_to_converged, r.timing['tc_spec_reruns'], r.timing['tc_speculated'], r.total_policy_evals,
              "equal to first:", bool((a == next(iter(res.values()))).all()), flush=True)
