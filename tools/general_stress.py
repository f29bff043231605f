"""Randomised stress of the general closed-form engine (PCD_ENGINE_GENERAL)
against the exact replay sweep (both on the GPU, one iteration each through
picard_iterate_once): random instances, plans (uniform, blocked, product-ish
with reassigned slots, single process), caches (garbage, serial trajectory
with perturbations, null), windows and feasible checkpoints.

  python tools/general_stress.py [cases] [seed]   -> prints failures, exit 1 on any
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = 0
for c in range(cases):
    J = int(rng.integers(1, 48))
    I = int(rng.integers(1, 120))
    T = int(rng.integers(1, 9000))
    inst = P.generate_instance(J, I, T, float(rng.choice([0.0, -0.5, -1.0])), float(rng.uniform(0.2, 1.0)),
                               int(rng.integers(1, 1 << 30)))
    kind = int(rng.integers(0, 3))
    pol = (P.GreedyPolicy() if kind == 0 else P.CapacityPenalizedPolicy(float(rng.uniform(0, 3))) if kind == 1
           else P.DualNetworkPolicy.seeded(inst, int(rng.integers(1, 100))))
    M = int(rng.integers(1, 300))
    style = int(rng.integers(0, 4))
    if style == 0:
        owner = P.make_uniform_time_partition(T, M, int(rng.integers(1, 1000))).owner
    elif style == 1:
        owner = np.minimum(np.arange(T) * M // max(T, 1), M - 1).astype(np.int32)
    elif style == 2:
        owner = P.make_product_partition(inst, M, 1).owner.copy()
        flip = rng.random(T) < 0.1
        owner[flip] = rng.integers(0, M, int(flip.sum()))
    else:
        M = 1
        owner = np.zeros(T, np.int32)
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
    plan = P.PartitionPlan(M, owner)
    outs = {}
    for e in ("replay", "general"):
        got = cache.copy()
        try:
            o = P.picard_iterate_once(inst, pol, plan, got, lo, hi, cap, inv, e)
            outs[e] = (got.tolist(), o.evals_per_process.tolist(), o.changed_slots.tolist())
        except P.ContractViolation as ex:
            outs[e] = ("ContractViolation", ex.time_step)
    if outs["replay"] != outs["general"]:
        bad += 1
        print("MISMATCH", dict(case=c, J=J, I=I, T=T, M=M, kind=kind, style=style, cstyle=cstyle, lo=lo, hi=hi),
              flush=True)
print(f"{cases} cases, {bad} mismatches", flush=True)
sys.exit(1 if bad else 0)
