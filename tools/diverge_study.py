"""Study (not a test): how many evaluations per Picard iteration follow a
process's first changed own slot ("diverged" suffixes). Before that slot a
process holds exactly the frozen-cache replay state, so its decisions there
equal a process-independent batch evaluation of every window slot.

  python tools/diverge_study.py J I T M product|chunk
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

J, I, T, M = (int(x) for x in sys.argv[1:5])
part = sys.argv[5]
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, M, 1) if part == "chunk" else P.make_product_partition(inst, M, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    r = sim.simulate(P.PicardConfig(record_trace=True, max_iterations=90), record_history=True)
H = r.history
owner = plan.owner
order = np.argsort(owner, kind="stable")  # slots grouped by process, time order
starts = np.searchsorted(owner[order], np.arange(M + 1))
prev = np.full(T, -1, np.int32)
tot_evals = tot_div = 0
rows = []
for k, row in enumerate(r.trace):
    lo = row.t_reset
    cur = H[k]
    ch = np.flatnonzero(cur[lo:] != prev[lo:]) + lo
    first = np.full(M, T, np.int64)
    np.minimum.at(first, owner[ch], ch)
    ev = 0
    div = 0
    # own slots in window per process and after its first change
    pos_lo = np.array([np.searchsorted(order[starts[m]:starts[m + 1]], 0) for m in range(0)])
    own_t = order  # slots sorted by (process, time)
    proc = owner[own_t]
    inwin = own_t >= lo
    ev = int(inwin.sum())
    div = int((inwin & (own_t >= first[proc])).sum())
    tot_evals += ev
    tot_div += div
    rows.append((k + 1, lo, len(ch), ev, div))
    prev = cur
for x in rows[:8] + rows[8::8]:
    print("it %3d lo %9d changed %8d evals %9d diverged %9d (%.3f)" % (*x, x[4] / max(1, x[3])))
print(f"TOTAL iterations {len(rows)} evals {tot_evals} diverged {tot_div} ({tot_div / tot_evals:.4f})")
