"""Small driver for ncu captures / phase profiles of the sweep kernels (not a test).

  python tools/tc_ncu_target.py J I T M [engine] [--cap] [--chunk]
"""
import sys

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

J, I, T, M = (int(x) for x in sys.argv[1:5])
engine = sys.argv[5] if len(sys.argv) > 5 and not sys.argv[5].startswith("--") else "product"
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, M, 1) if "--chunk" in sys.argv else P.make_product_partition(inst, M, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    cfg = P.PicardConfig(engine=engine, max_iterations=3 if "--cap" in sys.argv else 0)
    try:
        r = sim.simulate(cfg)
        print(r.iterations_to_converged, r.timing["sweep_ms"])
    except P.IterationLimitError as e:
        print("capped", e.iterations_run, sim.timing()["sweep_ms"])
