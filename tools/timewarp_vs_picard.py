"""Time Warp safe-window baseline vs the Picard fixed point on the device
(PAPER.md:288-292): same instance, policy and product
partition; sync rounds / iterations, the evaluation-speedup proxy
T / seq_equiv (theory.hpp:258-268) and device wall time.

  python tools/timewarp_vs_picard.py J I T M  -> JSON lines
"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

J, I, T, M = (int(x) for x in sys.argv[1:5])
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_partition(inst, M, 1)
t0 = time.perf_counter()
r = P.picard_simulate(inst, pol, plan, P.PicardConfig(max_steps=300 * M))
tp = time.perf_counter() - t0
print(json.dumps({"algo": "picard", "J": J, "I": I, "T": T, "M": M, "iterations": r.iterations_to_converged,
                  "seq_equiv": r.policy_eval_count_sequential_equivalent,
                  "proxy": T / r.policy_eval_count_sequential_equivalent, "wall_s": tp}), flush=True)
for rule in ("min_stocked_capacity", "min_capacity"):
    t0 = time.perf_counter()
    w = P.time_warp_simulate(inst, pol, M, 1, rule=rule)
    tw = time.perf_counter() - t0
    print(json.dumps({"algo": "time_warp", "rule": rule, "J": J, "I": I, "T": T, "M": M, "sync_rounds": w.sync_rounds,
                      "rollbacks": w.rollbacks, "seq_equiv": w.policy_eval_count_sequential_equivalent,
                      "proxy": T / w.policy_eval_count_sequential_equivalent, "wall_s": tw,
                      "same_actions_as_picard": bool((w.actions == r.actions).all())}), flush=True)
