"""Randomised stress of the tensor-core run-partition sweep (engine=product,
fp16x3 tcgen05 + FP64 margin recheck) against the exact FP64 engines, one
iteration each through picard_iterate_once: random instances (J up to the
tensor-core limit 103), product and product-chunk plans, dual-network
policies with random weight scales and normalisers, random caches (garbage,
perturbed serial trajectory, null), windows and feasible checkpoints.
Compares against engine=product_fp64 and engine=general.

  python tools/tc_stress.py [cases] [seed]   -> prints mismatches, exit 1 on any
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = tc_used = 0
for c in range(cases):
    J = int(rng.integers(1, 104))
    I = int(rng.integers(1, 200))
    T = int(rng.integers(1, 12000))
    inst = P.generate_instance(J, I, T, float(rng.choice([0.0, -0.5, -1.0])), float(rng.uniform(0.2, 1.0)),
                               int(rng.integers(1, 1 << 30)))
    params = P.MlpParams.seeded_uniform(2 * J + 1, 2 * J, int(rng.integers(1, 1000)))
    scale = float(rng.choice([0.5, 1.0, 1.0, 2.0]))
    for a in (params.w1, params.b1, params.w2, params.b2, params.w3, params.b3):
        a *= scale
    shrink = int(rng.choice([1, 1, 2]))
    pol = P.DualNetworkPolicy(params, np.maximum(np.asarray(inst.capacity) // shrink, 1),
                              np.asarray(inst.inventory) // shrink, inst.horizon, J)
    M = int(rng.integers(1, 400))
    plan = P.make_product_chunk_partition(inst, M, 1) if rng.random() < 0.5 else P.make_product_partition(inst, M, 1)
    seq = P.sequential_simulate(inst, pol).actions
    cstyle = int(rng.integers(0, 3))
    if cstyle == 0:
        cache = rng.integers(-3, J + 2, T).astype(np.int32)
    elif cstyle == 1:
        cache = seq.copy()
        flip = rng.random(T) < rng.uniform(0, 0.3)
        cache[flip] = rng.integers(-1, J, int(flip.sum()))
    else:
        cache = np.full(T, -1, np.int32)
    lo = int(rng.integers(0, T))
    hi = int(rng.integers(lo, T + 1))
    cap = np.array(inst.capacity, np.int32).copy()
    inv = np.array(inst.inventory, np.int32).reshape(I, J).copy()
    prod = np.array(inst.product)
    for t in range(lo):
        a = int(seq[t]) if rng.random() < 0.7 else int(rng.integers(-1, J))
        if a >= 0 and cap[a] > 0 and inv[prod[t], a] > 0:
            cap[a] -= 1
            inv[prod[t], a] -= 1
    outs = {}
    for e in ("product", "product_fp64", "general"):
        got = cache.copy()
        try:
            o = P.picard_iterate_once(inst, pol, plan, got, lo, hi, cap, inv, e)
            outs[e] = (got.tolist(), o.evals_per_process.tolist(), o.changed_slots.tolist())
        except P.ContractViolation as ex:
            outs[e] = ("ContractViolation", ex.time_step)
    # the tensor-core engine is taken when eligible; a full simulate reports it
    if c % 10 == 0:
        r = P.picard_simulate(inst, pol, plan, P.PicardConfig(engine="product", tc_verify=True))
        tc_used += r.timing["tc_used"]
        if r.timing["tc_unflagged_bad"] or r.actions.tolist() != seq.tolist():
            bad += 1
            print("VERIFY", dict(case=c, J=J, I=I, T=T, M=M, scale=scale, shrink=shrink), flush=True)
    if not (outs["product"] == outs["product_fp64"] == outs["general"]):
        bad += 1
        print("MISMATCH", dict(case=c, J=J, I=I, T=T, M=M, scale=scale, shrink=shrink, cstyle=cstyle, lo=lo, hi=hi),
              flush=True)
print(f"{cases} cases, {bad} mismatches, tensor-core path on {tc_used} of {(cases + 9) // 10} verified runs",
      flush=True)
sys.exit(1 if bad else 0)
