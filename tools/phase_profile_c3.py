"""Per-phase clock profile of the tensor-core sweep at C3 (PCD debug flag 1;
not a test): python tools/phase_profile_c3.py [window] [kernel...]"""
import sys
sys.path.insert(0, ".")
import paper_2406_01939_b200 as P
W = int(sys.argv[1]) if len(sys.argv) > 1 else 500000
inst = P.generate_instance(100, 10000, 10000000, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
plan = P.make_product_chunk_partition(inst, 65536, 1)
with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    P._capi.LIB.pcd_set_debug(sim._h, 1)
    for k in sys.argv[2:] or ["incremental"]:
        try:
            sim.simulate(P.PicardConfig(max_steps=W, tc_kernel=k, max_iterations=45))
        except P.IterationLimitError:
            pass
