"""Small driver for ncu captures / phase profiles of the sweep kernels (not a test).

  python tools/tc_ncu_target.py J I T M [engine] [--cap K] [--chunk | --wplan] [--window W] [--evals K]

--cap K    stop after K iterations (IterationLimitError is expected)
--evals K  also print the evaluations (all / tensor-core rows) of iteration K,
           from two capped runs (K-1 and K iterations), for per-launch units
"""
import sys

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402


def arg(name, default):
    return int(float(sys.argv[sys.argv.index(name) + 1])) if name in sys.argv else default


J, I, T, M = (int(x) for x in sys.argv[1:5])
engine = sys.argv[5] if len(sys.argv) > 5 and not sys.argv[5].startswith("--") else "product"
window = arg("--window", 0)
inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
pol = P.DualNetworkPolicy.seeded(inst, 5)
if "--wplan" in sys.argv:  # the bench's plan: window-aware chunks for this window
    plan = P.make_product_window_partition(inst, M, window, 1)
elif "--chunk" in sys.argv:
    plan = P.make_product_chunk_partition(inst, M, 1)
else:
    plan = P.make_product_partition(inst, M, 1)


def run(sim, cap):
    cfg = P.PicardConfig(engine=engine, max_steps=window, max_iterations=cap)
    try:
        r = sim.simulate(cfg)
        return "converged", r.iterations_to_converged, sim.timing()
    except P.IterationLimitError as e:
        return "capped", e.iterations_run, sim.timing()


with P.Simulator(inst, pol) as sim:
    sim.set_plan(plan)
    k = arg("--evals", 0)
    if k:
        _, _, a = run(sim, k - 1)
        _, _, b = run(sim, k)
        print(f"iteration {k}: evals {b['total_evals'] - a['total_evals']} "
              f"tc_rows {b['tc_rows'] - a['tc_rows']}")
    state, it, t = run(sim, arg("--cap", 0))
    print(state, it, t["sweep_ms"], t["total_ms"])
