"""Tuning helper (not a test): sweep time of the C3 fixed point vs tc_guard."""
import sys
import time

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

inst = P.generate_instance(100, 10000, 10_000_000, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, 65536, 1)
guards = [float(g) for g in sys.argv[1:]] or [5e-5]
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for g in guards:
        for rep in range(2):
            t0 = time.time()
            r = sim.simulate(P.PicardConfig(engine="product", tc_guard=g, max_steps=19_660_800))
            tm = r.timing
            print(f"guard={g:g} it={r.iterations_to_converged} total={1e3*(time.time()-t0):.1f}ms "
                  f"sweep={tm['sweep_ms']:.1f} prep={tm['prep_ms']:.1f} flagged={tm['tc_flagged']} "
                  f"tc_wrong_flagged={tm['tc_disagree']}", flush=True)
