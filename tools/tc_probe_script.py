"""GPU probe: FP64 vs tensor-core sweep timings and guard verification (not a test)."""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2406_01939_b200 as P  # noqa: E402

J, I, T, M = (int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (100, 1000, 1_000_000, 4096)))
verify = "--verify" in sys.argv
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_partition(inst, M, 1)
sim = P.Simulator(inst, pol)
sim.set_plan(plan)
keys = ("total_ms", "sweep_ms", "prep_ms", "advance_ms", "total_evals", "steps_critical", "tc_rows", "tc_flagged",
        "tc_disagree", "tc_unflagged_bad", "tc_tiles")
ref = sim.simulate(P.PicardConfig(engine="product_fp64"))
print("fp64", ref.iterations_to_converged, json.dumps({k: ref.timing[k] for k in keys}), flush=True)
if verify:
    for g in (1e-5, 1e-6):
        r = sim.simulate(P.PicardConfig(engine="product", tc_verify=True, tc_guard=g))
        print("verify", g, np.array_equal(r.actions, ref.actions), json.dumps({k: r.timing[k] for k in keys}), flush=True)
for g in (0.0, 0.0):
    r = sim.simulate(P.PicardConfig(engine="product", tc_guard=g))
    print("tc", g, np.array_equal(r.actions, ref.actions), r.iterations_to_converged,
          json.dumps({k: r.timing[k] for k in keys}), flush=True)
