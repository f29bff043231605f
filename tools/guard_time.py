"""Tuning helper (not a test): C3 fixed-point time vs the tensor-core guard
(0 = the derived guard of tc_error_bound), at the bench window.

  python tools/guard_time.py [window] [guard ...]
"""
import sys
import time

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
guards = [float(g) for g in sys.argv[2:]] or [0.0, 5e-5]
inst = P.generate_instance(100, 10000, 10_000_000, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
print("derived (B, guard):", P.tc_error_bound(inst, pol), flush=True)
plan = P.make_product_chunk_partition(inst, 65536, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for g in guards:
        for rep in range(2):
            t0 = time.time()
            r = sim.simulate(P.PicardConfig(tc_guard=g, max_steps=W))
            tm = r.timing
            print(f"guard={tm['tc_guard']:.3g} it={r.iterations_to_converged} total={1e3*(time.time()-t0):.1f}ms "
                  f"device={tm['total_ms']:.1f} sweep={tm['sweep_ms']:.1f} prep={tm['prep_ms']:.1f} "
                  f"rows={tm['tc_rows']} flagged={tm['tc_flagged']} ({100*tm['tc_flagged']/max(tm['tc_rows'],1):.3f}%) "
                  f"tc_wrong_flagged={tm['tc_disagree']} spec={tm.get('tc_speculated')} reruns={tm.get('tc_spec_reruns')}", flush=True)
