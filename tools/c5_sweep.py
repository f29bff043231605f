"""BASELINE.json configs[4] (C5): process-count sweep at fixed T = 10^7 on the C3
instance (J=100, I=10^4, dual MLP theta 5): iterations to convergence,
critical path and steps/s for product partitions (the reference's
partitioner; at most I processes carry work), product-chunk partitions and
(C5_PARTS=uniform) the reference's uniform time partition on the general
closed-form engine.

  [C5_PARTS=product,chunk,uniform] [C5_REPS=2] [C5_WINDOW=300000] python tools/c5_sweep.py [M ...]
  (C5_WINDOW: PicardConfig::max_steps; default the CLI's 300*M)
  -> one JSON line per (partition, M)
"""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

Ms = [int(x) for x in sys.argv[1:]] or [256, 1024, 4096, 16384, 65536]
J, I, T = 100, 10_000, 10_000_000
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
seq = None
PARTS = os.environ.get("C5_PARTS", "product,chunk").split(",")
REPS = int(os.environ.get("C5_REPS", "2"))
WINDOW = int(os.environ.get("C5_WINDOW", "0"))
for part in PARTS:
    for M in Ms:
        if part == "chunk":
            plan = P.make_product_chunk_partition(inst, M, 1)
        elif part == "uniform":
            plan = P.make_uniform_time_partition(T, M, 1)
        else:
            plan = P.make_product_partition(inst, M, 1)
        with P.Simulator(inst, pol) as sim:
            sim.set_plan(plan)
            cfg = P.PicardConfig(max_steps=WINDOW or 300 * M)
            r = sim.simulate_resident(cfg)  # warm-up (the timed run when REPS = 0)
            best = r.timing["total_ms"] if REPS == 0 else None
            for _ in range(REPS):
                r = sim.simulate_resident(cfg)
                ms = r.timing["total_ms"]
                best = ms if best is None else min(best, ms)
            acts = sim.download_actions()
        if seq is None:
            seq = acts
        print(json.dumps({"config": "c5", "partition": part, "M": M, "max_steps": WINDOW or 300 * M,
                          "engine_used": r.timing["engine_used"], "tc_flagged": r.timing["tc_flagged"],
                          "iterations": r.iterations_to_converged,
                          "steps_critical": r.timing["steps_critical"], "total_evals": r.total_policy_evals,
                          "ms": best, "steps_per_s": T / (best / 1000.0),
                          "same_trajectory": bool((acts == seq).all())}), flush=True)
