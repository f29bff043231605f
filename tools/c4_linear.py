"""BASELINE.json configs[3] (C4): the non-SCO env of the reference
(linear::make_contractive_spec n=4, p=4, rho, GainPolicy) under single-step
Picard partitions (M = T): iterations to tolerance vs horizon, device time of
the B200 affine-scan engine, and the reference's picard_convergence_curve
(oracle/_ref, 1 core; O(T^2) per iteration) timed where it finishes.

  python tools/c4_linear.py  -> JSON lines
"""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402
from oracle.oracle import REF  # noqa: E402

rho, tol = 0.5, 1e-6
for T in (1_000, 10_000, 100_000, 1_000_000):
    for coupling in ((0.0, 0.3) if T <= 100_000 else (0.0,)):  # coupled specs: host bisection per step
        spec = P.make_contractive_spec(4, 4, T, rho, 7, coupling)
        P.picard_convergence_curve(spec, tolerance=tol)  # warm-up
        t0 = time.perf_counter()
        r = P.picard_convergence_curve(spec, tolerance=tol)
        wall = time.perf_counter() - t0
        line = {"config": "c4", "T": T, "n": 4, "p": 4, "rho": rho, "state_coupling": coupling, "tolerance": tol,
                "iterations": int(r.curve.size), "final_rmse": float(r.curve[-1]), "device_ms": r.device_ms,
                "wall_ms": 1e3 * wall, "steps_per_s": T * r.curve.size / (r.device_ms / 1e3)}
        if T <= 2_000:
            t1 = time.perf_counter()
            want = REF.linear_curve(spec, tolerance=tol)
            line["reference_s"] = time.perf_counter() - t1
            line["reference_iterations"] = int(want.size)
            line["max_rel_diff"] = float(np.max(np.abs(r.curve - want) / np.maximum(np.abs(want), 1e-300)))
        print(json.dumps(line), flush=True)
