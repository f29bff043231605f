"""A/B of the two tensor-core sweeps (fused layer 1 vs incremental layer 1):
identical trajectories and counters, times (not a test; tests/ cover parity).

  python tools/inc_check.py [--c3] [--prof]
"""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2406_01939_b200 as P  # noqa: E402

CASES = [(10, 60, 3000, 32, "product", 0), (10, 60, 3000, 64, "chunk", 0), (30, 400, 40000, 512, "chunk", 5000),
         (100, 300, 30000, 512, "chunk", 0), (10, 1000, 1000000, 4096, "chunk", 0)]
if "--c3" in sys.argv:
    CASES.append((100, 10000, 10000000, 65536, "chunk", 500000))

for J, I, T, M, part, window in CASES:
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    plan = (P.make_product_chunk_partition(inst, M, 1) if part == "chunk" else P.make_product_partition(inst, M, 1))
    out = {}
    with P.Simulator(inst, pol) as sim:
        sim.set_plan(plan)
        if "--prof" in sys.argv:
            P._capi.LIB.pcd_set_debug(sim._h, 1)
        for kern in ("fused", "incremental", "fused", "incremental"):
            cfg = P.PicardConfig(max_steps=window, tc_kernel=kern)
            t0 = time.time()
            r = sim.simulate(cfg)
            wall = time.time() - t0
            tm = sim.timing()
            out[kern] = (r, tm)
            print(f"J={J} I={I} T={T} M={M} {part} W={window} {kern:11s}: it={r.iterations_to_converged} "
                  f"evals={r.total_policy_evals} sweep={tm['sweep_ms']:.2f} ms total={tm['total_ms']:.2f} ms "
                  f"wall={wall*1e3:.1f} ms tc_kernel={tm['tc_kernel']} inc_iters={tm['tc_inc_iters']} "
                  f"flagged={tm['tc_flagged']} dis={tm['tc_disagree']}", flush=True)
    a, b = out["fused"][0], out["incremental"][0]
    same = (np.array_equal(a.actions, b.actions) and a.iterations_to_converged == b.iterations_to_converged
            and a.conflicts == b.conflicts and a.total_policy_evals == b.total_policy_evals)
    print("  same trajectory and counters:", same, flush=True)
    assert same
