"""How much a window's states move between two Picard iterations at C3 (not a
test): from the cache after each of the first 45 iterations, for slots t of
iteration k+2's window, the number N of effective-action changes before t
between the inputs of iterations k+1 and k+2, and the net per-node capacity
change sum_j |dF_j(t)| and max_j |dF_j(t)|. Evidence for DESIGN.md §7
(certified reuse of decisions across iterations: rejected).
  python tools/iteration_drift.py > profiles/r02_iteration_drift.txt
"""
import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np
import paper_2406_01939_b200 as P
from paper_2406_01939_b200._capi import LIB
W = 300000
inst = P.generate_instance(100, 10000, 10_000_000, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, 65536, 1)
T = 10_000_000; K = 45
hist = np.zeros((K, T), np.int32)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    LIB.pcd_set_history(sim._h, hist.ctypes.data_as(C.POINTER(C.c_int)), K)
    r = sim.simulate(P.PicardConfig(max_steps=W, record_trace=True))
    LIB.pcd_set_history(sim._h, None, 0)
ws = [row.t_reset for row in r.trace]
print("iterations", len(ws), ws[:12])
J = 100
for k in range(5, K - 1, 4):
    # iteration k+1 (1-based) has input hist[k-1]; iteration k+2 has input hist[k]
    a, b = hist[k - 1], hist[k]
    lo0, lo1 = ws[k], ws[k + 1]  # windows of iterations k+1 and k+2 (0-based trace rows k, k+1)
    reg = slice(lo0, min(T, lo1 + W))
    d = np.nonzero(a[reg] != b[reg])[0] + lo0
    if len(d) == 0:
        continue
    old, new = a[d], b[d]
    M = np.zeros((len(d), J), np.int32)
    ok = old >= 0; M[np.nonzero(ok)[0], old[ok]] -= 1
    ok = new >= 0; M[np.nonzero(ok)[0], new[ok]] += 1
    cum = np.cumsum(M, axis=0)
    ts = np.arange(lo1, min(T, lo1 + W), 5000)
    idx = np.searchsorted(d, ts)  # changes before t
    n = idx
    net = np.array([np.abs(cum[i - 1]).sum() if i > 0 else 0 for i in idx])
    mx = np.array([np.abs(cum[i - 1]).max() if i > 0 else 0 for i in idx])
    q = lambda x: np.percentile(x, [10, 50, 90]).astype(int).tolist()
    print(f"it {k+2}: window lo {lo1}, changed in prev {len(d)}; 2N q10/50/90 {q(2*n)}  net sum|dF| {q(net)}  max|dF_j| {q(mx)}", flush=True)
