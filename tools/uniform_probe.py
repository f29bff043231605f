import sys, time
sys.path.insert(0, ".")
import paper_2406_01939_b200 as P
for (J, I, T, M) in [(10, 1000, 100000, 256), (10, 1000, 1000000, 1024)]:
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, 5)
    plan = P.make_uniform_time_partition(T, M, 1)
    t0 = time.time()
    try:
        r = P.picard_simulate(inst, pol, plan, P.PicardConfig(max_steps=300 * M, max_iterations=5))
        print(J, I, T, M, "iters", r.iterations_to_converged, time.time() - t0, flush=True)
    except P.IterationLimitError as e:
        print(J, I, T, M, "capped at", e.iterations_run, "in", time.time() - t0, "s", flush=True)
