"""BASELINE.json configs[3] (C4) with an MLP policy: the reference's linear env
(make_contractive_spec n=4, p=4) under the MLP feedback policy a = forward(s)
(the reference's MlpParams {4, 64, 64, 4}, seeded, output layer scaled), single-
step Picard partitions (M = T). Per horizon: iterations to tolerance (the
curve), picard_simulate's iterations_to_converged, device time; the reference
(oracle/_ref: picard_convergence_curve restated with the MLP policy, and
picard_simulate with M = T, 1 core) where it finishes.

  python tools/c4_mlp.py  -> JSON lines
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402
from oracle.oracle import REF  # noqa: E402

tol = 1e-6
for rho, coupling, scale in ((0.5, 0.0, 20.0), (0.9, 0.5, 40.0)):
    for T in (1_000, 10_000, 100_000, 1_000_000):
        if coupling and T > 100_000:
            continue  # coupled specs: the generator's host bisection per step
        spec = P.make_contractive_spec(4, 4, T, rho, 7, coupling)
        pol = P.MlpFeedbackPolicy.seeded(4, 4, 3, 64, scale)
        P.picard_convergence_curve(spec, tolerance=tol, policy=pol)  # warm-up
        t0 = time.perf_counter()
        r = P.picard_convergence_curve(spec, tolerance=tol, policy=pol)
        wall = time.perf_counter() - t0
        line = {"config": "c4-mlp", "T": T, "n": 4, "p": 4, "hidden": 64, "rho": rho, "state_coupling": coupling,
                "output_scale": scale, "tolerance": tol, "curve_iterations": int(r.curve.size),
                "final_rmse": float(r.curve[-1]), "iterations_to_converged": r.iterations_to_converged,
                "fixed_point_iterations": r.fixed_point_iterations, "fixed_point_ms": r.fixed_point_ms,
                "device_ms": r.device_ms, "wall_ms": 1e3 * wall,
                "policy_evals_per_s": T * (r.fixed_point_iterations + r.curve.size) / (r.device_ms / 1e3)}
        if T <= 1_000:
            t1 = time.perf_counter()
            want = REF.linear_mlp_curve(spec, pol.params, tolerance=tol)
            line["reference_curve_s"] = time.perf_counter() - t1
            line["reference_curve_iterations"] = int(want.size)
            line["max_rel_diff"] = float(np.max(np.abs(r.curve - want) / np.maximum(np.abs(want), 1e-300)))
            t1 = time.perf_counter()
            it, _ = REF.linear_mlp_picard(spec, pol.params)
            line["reference_picard_s"] = time.perf_counter() - t1
            line["reference_iterations_to_converged"] = it
        print(json.dumps(line), flush=True)
