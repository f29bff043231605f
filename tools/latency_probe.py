"""Single-row latency of the tensor-core sweeps (not a test): one product and
one process, windows of W slots, so one row of one CTA steps through <= W own
slots per iteration. Prints the sweep time per step for both kernels.

  python tools/latency_probe.py [J] [T] [W] [iterations] [kernel...]
"""
import sys

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

J = int(sys.argv[1]) if len(sys.argv) > 1 else 100
T = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
W = int(sys.argv[3]) if len(sys.argv) > 3 else 100
NIT = int(sys.argv[4]) if len(sys.argv) > 4 else 40
TILES = 1
kerns = sys.argv[5:] or ["fused", "incremental", "fused", "incremental"]
inst = P.generate_instance(J, 1, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_partition(inst, 1, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for kern in kerns:
        try:
            sim.simulate(P.PicardConfig(tc_kernel=kern, max_steps=W, max_iterations=NIT, tc_tiles=TILES))
        except P.IterationLimitError:
            pass
        tm = sim.timing()
        print(f"{kern:11s} it={tm['iterations']} evals={tm['total_evals']} sweep={tm['sweep_ms']:.2f} ms "
              f"-> {1e3 * tm['sweep_ms'] / max(1, tm['total_evals']):.2f} us/step", flush=True)
