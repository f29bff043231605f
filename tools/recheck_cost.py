"""Tuning helper (not a test): cost of the exact FP64 re-evaluation per flagged
row, from sweep time with every row flagged (huge guard) vs the default."""
import sys
import time

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

J, I, T, M = 100, 400, 200000, 2400
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, M, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for g in (5e-5, 1e9, 5e-5, 1e9):
        r = sim.simulate(P.PicardConfig(engine="product", tc_guard=g, max_iterations=3))  if False else None
        try:
            r = sim.simulate(P.PicardConfig(engine="product", tc_guard=g))
            tm = r.timing
        except P.IterationLimitError:
            tm = sim.timing()
        print(f"guard={g:g} sweep={tm['sweep_ms']:.2f}ms rows={tm['tc_rows']} flagged={tm['tc_flagged']} "
              f"steps_critical={tm['steps_critical']} iters={tm['iterations']}", flush=True)
