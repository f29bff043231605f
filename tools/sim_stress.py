"""Randomised stress of picard_simulate end to end (the tensor-core sweep with
speculation and the pipelined verification, engine=auto) against the CPU
oracle's picard_simulate restatement (oracle/picard_oracle.c, engine.hpp:
458-590): random instances (J even, up to 100, so speculation applies),
product / equal-chunk / window-aware plans, random windows, random weight
scales, and the debug modes that force rejected speculation (every
speculated iteration re-run, or planted wrong decisions that the
verification must catch). Actions, iterations to converged / correct,
conflicts, evaluation counters and every trace row must equal the oracle's.

  python tools/sim_stress.py [cases] [seed]   -> prints mismatches, exit 1 on any
"""
import sys
from types import SimpleNamespace as NS

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402
from oracle.oracle import ORC  # noqa: E402
from tests.helpers import product_instance  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
bad = spec_cases = reruns = 0
for c in range(cases):
    J = 2 * int(rng.integers(1, 51))
    I = int(rng.integers(1, 300))
    T = int(rng.integers(100, 20000))
    ons = NS(**ORC.generate_instance_arrays(J, I, T, float(rng.choice([0.0, -0.5])), float(rng.uniform(0.3, 1.0)),
                                            int(rng.integers(1, 1 << 30)), geometry=0 if J <= 30 else 1))
    inst = product_instance(ons)
    p = P.MlpParams.seeded_uniform(2 * J + 1, 2 * J, int(rng.integers(1, 1000)))
    scale = float(rng.choice([0.5, 1.0, 2.0]))
    for a in (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3):
        a *= scale
    pol = P.DualNetworkPolicy(p, None, None, inst.horizon, J)
    opol = NS(kind=2, hidden=64, gamma=0.0, horizon=None, w1=pol.w1, b1=pol.b1, w2=pol.w2, b2=pol.b2,
              w3=pol.w3, b3=pol.b3)
    M = int(rng.integers(1, 1200))
    W = int(rng.choice([0, int(rng.integers(50, max(51, T)))]))
    part = rng.choice(["window", "chunk", "product"])
    plan = (P.make_product_window_partition(inst, M, W, 1) if part == "window"
            else P.make_product_chunk_partition(inst, M, 1) if part == "chunk" else P.make_product_partition(inst, M, 1))
    flags = int(rng.choice([0, 0, 16, 32]))
    seq, _ = ORC.sequential(ons, opol)
    want = ORC.picard(ons, opol, plan.owner, M, max_steps=W, record_trace=True, reference=seq)
    with P.Simulator(inst, pol) as sim:
        sim.set_plan(plan)
        P._capi.LIB.pcd_set_debug(sim._h, flags)
        got = sim.simulate(P.PicardConfig(max_steps=W, record_trace=True), reference_actions=seq)
    t = got.timing
    spec_cases += t["tc_speculated"] > 0
    reruns += t["tc_spec_reruns"]
    ok = (np.array_equal(got.actions, seq) and got.iterations_to_converged == want.iterations_to_converged
          and got.iterations_to_correct == want.iterations_to_correct and got.conflicts == want.conflicts
          and got.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent
          and got.total_policy_evals == want.total_policy_evals
          and [x.astuple() for x in got.trace] == [tuple(x) for x in want.trace])
    if not ok:
        bad += 1
        print(f"MISMATCH case {c}: J={J} I={I} T={T} M={M} W={W} plan={part} flags={flags} "
              f"iters {got.iterations_to_converged}/{want.iterations_to_converged}", flush=True)
print(f"{cases} cases, {bad} mismatches; {spec_cases} with speculated decisions, {reruns} rejected "
      f"speculations re-run", flush=True)
sys.exit(1 if bad else 0)
