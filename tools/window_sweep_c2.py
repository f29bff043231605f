"""C2 (J=10, I=1e3, T=1e6, M=4096) window-width sweep; see window_sweep.py."""
import json
import sys

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

Ws = [int(float(x)) for x in sys.argv[1:]] or [0, 300_000, 100_000, 30_000, 10_000]
J, I, T, M = 10, 1000, 1_000_000, 4096
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
for part in ("chunk", "product"):
    plan = P.make_product_chunk_partition(inst, M, 1) if part == "chunk" else P.make_product_partition(inst, M, 1)
    seq = None
    with P.Simulator(inst, pol) as sim:
        sim.set_plan(plan)
        for W in Ws:
            cfg = P.PicardConfig(max_steps=W)
            sim.simulate_resident(cfg)
            r = sim.simulate_resident(cfg)
            acts = sim.download_actions()
            seq = acts if seq is None else seq
            t = r.timing
            print(json.dumps({"config": "c2", "max_steps": W, "partition": part, "iterations": r.iterations_to_converged,
                              "total_evals": r.total_policy_evals, "steps_critical": t["steps_critical"],
                              "ms": t["total_ms"], "sweep_ms": t["sweep_ms"], "prep_ms": t["prep_ms"],
                              "advance_ms": t["advance_ms"], "same_trajectory": bool((acts == seq).all())}), flush=True)
