"""Per-phase clock profile of the tensor-core sweep at C3 (PCD debug flag 1;
not a test): python tools/phase_profile_c3.py [window] [guard] [iterations]
(guard 0 = the derived guard; PP_PLAN=window: the window-aware plan). Prints one tcprof line per iteration (CTA 0,
half 0) and the column sums over the run."""
import re
import sys

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 500000
G = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
N = int(sys.argv[3]) if len(sys.argv) > 3 else 45
inst = P.generate_instance(100, 10000, 10000000, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
import os  # noqa: E402
plan = (P.make_product_window_partition(inst, 65536, W, 1) if os.environ.get("PP_PLAN") == "window"
        else P.make_product_chunk_partition(inst, 65536, 1))
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    P._capi.LIB.pcd_set_debug(sim._h, 1)
    try:
        sim.simulate(P.PicardConfig(max_steps=W, tc_guard=G, tc_kernel="fused", max_iterations=N))
    except P.IterationLimitError:
        pass
