"""Window width x partition sweep on the C3 instance: for each window W
(PicardConfig::max_steps, engine.hpp:120-126) the window-aware product chunks
(make_product_window_partition(M, W)) next to the equal-count chunks
(make_product_chunk_partition(M)). Every run must reach the same trajectory
(Prop. 1); the window-aware plan bounds each iteration's per-process chain.

  python tools/window_partition_sweep.py [W ...]      (default 200k 300k 400k)
  WS_M=65536  WS_PARTS=window,chunk  WS_SHAPE=J,I,T (default the C3 shape 100,10000,1e7)
  -> one JSON line per (window, partition); ms = best of two resident runs
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

Ws = [int(float(x)) for x in sys.argv[1:]] or [200_000, 300_000, 400_000]
J, I, T = (int(float(x)) for x in os.environ.get("WS_SHAPE", "100,10000,1e7").split(","))  # C2: 10,1000,1e6
M = int(os.environ.get("WS_M", "65536"))
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
seq = None
with P.Simulator(inst, pol) as sim:
    for W in Ws:
        for part in os.environ.get("WS_PARTS", "window,chunk").split(","):
            plan = (P.make_product_window_partition(inst, M, W, 1) if part == "window"
                    else P.make_product_chunk_partition(inst, M, 1))
            own = np.asarray(plan.owner)
            sim.set_plan(plan)
            cfg = P.PicardConfig(max_steps=W)
            best = None
            for _ in range(3):
                r = sim.simulate_resident(cfg)
                if best is None or r.timing["total_ms"] < best.timing["total_ms"]:
                    best = r
            acts = sim.download_actions()
            if seq is None:
                seq = acts
            t = best.timing
            print(json.dumps({"max_steps": W, "M": M, "partition": part, "processes_used": int(own.max()) + 1,
                              "iterations": best.iterations_to_converged, "total_evals": best.total_policy_evals,
                              "steps_critical": t["steps_critical"], "ms": t["total_ms"], "sweep_ms": t["sweep_ms"],
                              "prep_ms": t["prep_ms"], "advance_ms": t["advance_ms"],
                              "steps_per_s": T / (t["total_ms"] / 1e3), "spec_reruns": t.get("tc_spec_reruns"),
                              "same_trajectory": bool((acts == seq).all())}), flush=True)
