"""C3 on the exact FP64 SIMT engines (not a test): the run-partition sweep
(engine=product_fp64) and the general closed form (engine=general) on the
product-chunk plan, same trajectory as the tensor-core sweep. One JSON line
per engine (profiles/r01_fp64_engines_c3.jsonl).

  python tools/fp64_engines_probe.py
"""
import sys, json
sys.path.insert(0, ".")
import paper_2406_01939_b200 as P
J, I, T, M = 100, 10_000, 10**7, 65536
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, M, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for eng in ("product_fp64", "general"):
        r = sim.simulate_resident(P.PicardConfig(max_steps=300 * M, engine=eng))
        tm = r.timing
        print(json.dumps(dict(engine=eng, it=r.iterations_to_converged, ms=tm["total_ms"], sweep=tm["sweep_ms"],
                              prep=tm["prep_ms"], evals=r.total_policy_evals)), flush=True)
