"""Window-width (PicardConfig::max_steps, engine.hpp:120-126) sweep on the C3
instance: any window reaches the same serial trajectory (Prop. 1; window-width
invariance, test_engine.cpp:455-477), but the evaluations per iteration and
the iteration count depend on it.

  python tools/window_sweep.py [max_steps ...]   (0 = whole horizon)
  WS_M=65536 WS_PART=chunk
  -> one JSON line per window
"""
import json
import os
import sys

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

Ws = [int(float(x)) for x in sys.argv[1:]] or [0, 3_000_000, 1_000_000, 300_000, 100_000]
J, I, T = 100, 10_000, 10_000_000
M = int(os.environ.get("WS_M", "65536"))
part = os.environ.get("WS_PART", "chunk")
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, M, 1) if part == "chunk" else P.make_product_partition(inst, M, 1)
seq = None
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    for W in Ws:
        cfg = P.PicardConfig(max_steps=W)
        sim.simulate_resident(cfg)
        r = sim.simulate_resident(cfg)
        acts = sim.download_actions()
        if seq is None:
            seq = acts
        t = r.timing
        print(json.dumps({"max_steps": W, "M": M, "partition": part, "iterations": r.iterations_to_converged,
                          "total_evals": r.total_policy_evals, "steps_critical": t["steps_critical"],
                          "ms": t["total_ms"], "sweep_ms": t["sweep_ms"], "prep_ms": t["prep_ms"],
                          "advance_ms": t["advance_ms"], "steps_per_s": T / (t["total_ms"] / 1e3),
                          "same_trajectory": bool((acts == seq).all())}), flush=True)
