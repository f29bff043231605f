"""Tuning helper (not a test): wall-clock breakdown of the one-shot public API
(pcd_create / pcd_set_plan / pcd_simulate incl. download / pcd_destroy)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2406_01939_b200 as P  # noqa: E402
from bench import default_window, make_workload  # noqa: E402

inst, pol, plan, w = make_workload("c3", sys.argv[1] if len(sys.argv) > 1 else "chunk")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
pinst = P.Instance(inst.nodes, inst.products, inst.horizon, pin(inst.product), pin(inst.reward_row),
                   pin(inst.reward_table), pin(inst.capacity), pin(inst.inventory))
pplan = P.PartitionPlan(plan.processes, pin(plan.owner))
cfg = P.PicardConfig(max_steps=default_window("c3"))
for rep in range(3):
    t0 = time.perf_counter()
    sim = P.Simulator(pinst, pol)
    t1 = time.perf_counter()
    sim.set_plan(pplan)
    t2 = time.perf_counter()
    r = sim.simulate(cfg)
    t3 = time.perf_counter()
    sim.close()
    t4 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} set_plan {1e3*(t2-t1):.1f} simulate {1e3*(t3-t2):.1f} "
          f"(engine {r.timing['total_ms']:.1f}) destroy {1e3*(t4-t3):.1f} total {1e3*(t4-t0):.1f} ms", flush=True)
for rep in range(3):
    t0 = time.perf_counter()
    r = P.picard_simulate(pinst, pol, pplan, cfg)
    t1 = time.perf_counter()
    print(f"one-shot picard_simulate {1e3*(t1-t0):.1f} ms (engine {r.timing['total_ms']:.1f})", flush=True)
