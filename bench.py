#!/usr/bin/env python3
"""bench.py — simulated time-steps/s to convergence of ONE trajectory
(BASELINE.json "metric"), B200 Picard engine vs the reference's CPU paths.

Workload (default "c3", BASELINE.json configs[2], the north-star target and the
largest config; it fits one B200): SCO with J=100 nodes, I=10^4 products,
T=10^7 orders (generate_instance recipe, seed 7, beta 0, coverage 0.8, the
seeded synthetic 100-node geometry), dual-price MLP policy {201,64,64,200}
with theta seed 5, M=65536 processes, max_steps = 350,000 (the window; the
CLI default 300*M = the whole horizon is timed beside it, same trajectory).
Partition (--partition): "window" (default) =
make_product_window_partition(M, max_steps): every product's orders cut into
contiguous chunks, one process each, so that no window of max_steps orders
holds more than L orders of one process (L minimal for <= M chunks: 44 at the
C3 window of 350k, where equal chunks leave ~58); "chunk" =
make_product_chunk_partition(M): equal-count contiguous chunks; "product" = the
reference's make_product_partition(M, seed 1), which activates only I=10^4 of
them. All reach the same (serial) trajectory. One "step" = one full
picard_simulate to convergence. Synthetic data, random-init weights.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload c3|c2|c1]

N>1 runs under torchrun, one rank per GPU: processes are sharded over ranks and
every iteration exchanges fresh cache slices with NCCL (strong scaling of one
trajectory). Timing: CUDA events around exactly K steps, barrier+sync on both
sides, max over ranks. The L2 (126 MB) is flushed with a 512 MiB write before
every step; the working set (orders 80 MB, cache 40 MB, ...) exceeds L2 anyway.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (J, I, T, M, theta seed) — BASELINE.json configs
    "c1": (1, 10, 10_000, 16, 5),
    "c2": (10, 1_000, 1_000_000, 4096, 5),
    "c3": (100, 10_000, 10_000_000, 65536, 5),
}
# PicardConfig::max_steps (the window, engine.hpp:120-126, :529-531) per
# workload. Every window reaches the same serial trajectory (Prop. 1; the
# reference's window-width invariance test, test_engine.cpp:455-477); the
# width only changes how much of the horizon each iteration re-evaluates.
# C3: 350,000 with the window-aware plan cut for it
# (profiles/r02_window_partition_sweep_c3.jsonl: 73.6 ms vs 75.0 at 300k,
# 73.8 at 400k, 77.2 at 500k, 93 at 1M; the CLI default 300*M is the whole
# horizon here); C2/C1: the CLI default (cli.cpp:225-227), narrower windows
# are slower there.
WINDOWS = {"c1": None, "c2": None, "c3": 350_000}


def default_window(name: str) -> int:
    M = WORKLOADS[name][3]
    return WINDOWS[name] if WINDOWS[name] is not None else 300 * M
METRIC = "simulated time-steps/sec to convergence (1 trajectory); speedup vs serial CPU ref"
PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")


def flops_per_eval(J: int, H: int = 64) -> int:
    """Algorithmic FLOPs of one dual-policy evaluation: the three GEMV layers of
    MlpParams::forward (mlp.cpp:141-169), 2 per MAC."""
    return 2 * (H * (2 * J + 1) + H * H + 2 * J * H)


def load_peaks():
    try:
        with open(PEAKS) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons sampled during the timed region through NVML
    (in-process, every 0.2 s; nvidia-smi's CLI is the fallback: forking it every
    sample adds host stalls to the measured region)."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4))
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.index = index
        self.enabled = enabled
        self.rows = []  # (sm_mhz, max_mhz, [reason names])
        self._stop = threading.Event()
        self._t = None
        self._nv = None
        try:
            import pynvml
            pynvml.nvmlInit()
            h = None
            try:
                import torch
                bus = torch.cuda.get_device_properties(index).pci_bus_id
                pci = f"00000000:{bus:02x}:00.0"
                h = pynvml.nvmlDeviceGetHandleByPciBusId(pci)
            except Exception:
                h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nv = (pynvml, h)
        except Exception:
            self._nv = None

    def _sample(self):
        if self._nv:
            nv, h = self._nv
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            try:
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            except Exception:
                bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            return float(sm), float(mx), [n for n, b in self.REASONS if bits & b]
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        r = [x.strip() for x in out.split(",")]
        names = [n for n, _ in self.REASONS]
        return (float(r[0]), float(r[1]), [n for n, v in zip(names, r[3:7]) if v.lower() == "active"])

    def _run(self):
        while self.enabled and not self._stop.is_set():
            try:
                self.rows.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({n for r in self.rows for n in r[2]}), "samples": len(self.rows),
                "source": "nvml" if self._nv else "nvidia-smi"}


PARTITIONS = {
    "product": "make_product_partition(M, seed 1) (the reference's partitioner)",
    "chunk": "make_product_chunk_partition(M): each product's orders cut into contiguous chunks, one process each",
    "window": "make_product_window_partition(M, max_steps): each product's orders cut into contiguous chunks so "
              "that no max_steps-long interval holds more than L orders of one chunk, L minimal for <= M chunks",
}
DTYPE = ("f64 decisions (fp16x3 tcgen05 MLP; rows whose decision margin is within the derived error bound "
         "2B are re-evaluated in exact FP64)")
NCU_PROFILE = os.path.join("profiles", "r02_ncu_sweep_pp_wplan.json")  # ncu --set full of the sweep (tools/ncu_summary.py)


def workload_config(args, world: int) -> dict:
    """The config dict both arms print (identical by construction)."""
    J, I, T, M, theta = WORKLOADS[args.workload]
    return {"workload": args.workload, "J": J, "I": I, "T": T, "M": M, "theta": theta,
            "policy": "dual MLP {2J+1,64,64,2J} seeded", "instance": "generate_instance(J, I, T, beta 0, "
            "coverage 0.8, seed 7)" + (", seeded synthetic J-node geometry" if J > 30 else ""),
            "partition": PARTITIONS[args.partition],
            "max_steps": default_window(args.workload) if args.max_steps is None else args.max_steps,
            "cli_default_max_steps": 300 * M,
            "l2": "512 MiB flush before every GPU step; working set > L2",
            "parallelism": f"processes sharded over {world} GPU(s)"}


def trajectory_hash(actions) -> str:
    """blake2b-64 of the int32 action array: both arms print it, so the same
    trajectory shows the same hash."""
    import hashlib
    return hashlib.blake2b(np.ascontiguousarray(actions, np.int32).tobytes(), digest_size=8).hexdigest()


def make_workload(name: str, partition: str = "product", window: int = 0):
    import paper_2406_01939_b200 as P
    J, I, T, M, theta = WORKLOADS[name]
    inst = P.generate_instance(J, I, T, 0.0, 0.8, 7)
    pol = P.DualNetworkPolicy.seeded(inst, theta)
    if partition == "window":
        plan = P.make_product_window_partition(inst, M, window or default_window(name), 1)
    elif partition == "chunk":
        plan = P.make_product_chunk_partition(inst, M, 1)
    else:
        plan = P.make_product_partition(inst, M, 1)
    return inst, pol, plan, dict(J=J, I=I, T=T, M=M, theta=theta)


def ref_workload(name: str):
    """The workload built through the CPU oracle only (the reference's own
    generate_instance / MlpParams::seeded_uniform via oracle/_ref, or the C
    restatement when the reference build is absent) — the reference arm never
    imports the product package."""
    from types import SimpleNamespace as NS
    from oracle.oracle import REF, ORC
    lib, kind = (REF, "reference") if REF is not None else (ORC, "port")
    J, I, T, M, theta = WORKLOADS[name]
    inst = NS(**lib.generate_instance_arrays(J, I, T, 0.0, 0.8, 7, geometry=0 if J <= 30 else 1))
    w = lib.seeded_mlp(2 * J + 1, 2 * J, theta)
    pol = NS(kind=2, hidden=64, gamma=0.0, horizon=T, w1=w[0], b1=w[1], w2=w[2], b2=w[3], w3=w[4], b3=w[5])
    return inst, pol, lib, kind


def oracle_policy_of(pol, T):
    from types import SimpleNamespace as NS
    return NS(kind=2, hidden=pol.hidden, gamma=0.0, horizon=T, w1=pol.w1, b1=pol.b1, w2=pol.w2, b2=pol.b2,
              w3=pol.w3, b3=pol.b3)


def state_at(inst, actions, t):
    """FoState after orders [0, t) of a trajectory (fo_transition applied in
    order; env.hpp / types.hpp:89-100): capacities and dense inventory."""
    a = np.asarray(actions[:t])
    ok = a >= 0
    J = int(inst.nodes)
    cap = np.asarray(inst.capacity, np.int64) - np.bincount(a[ok], minlength=J)[:J]
    inv = np.asarray(inst.inventory, np.int64).reshape(-1, J).copy()
    np.subtract.at(inv, (np.asarray(inst.product[:t])[ok], a[ok]), 1)
    return cap.astype(np.int32), inv.astype(np.int32).ravel()


def cpu_baseline(inst, pol, actions, budget_s: float = 20.0, segments: int = 8):
    """The UNMODIFIED reference's sequential_simulate (oracle/_ref), 1 host
    core (the serial path cannot use more), on a STRATIFIED sample of the
    same workload: `segments` equal stretches of n orders starting at
    k*T/segments, each started from the exact state the trajectory reaches
    there (the reference's actions on every stretch are compared with ours:
    equal stretches mean equal states). The horizon's tail is mostly
    declines (no forward pass, policies.hpp:127-134), so a head prefix would
    overstate the serial cost; the stratified sample does not."""
    from oracle.oracle import REF, ORC
    T = int(inst.horizon)
    opol = oracle_policy_of(pol, T)
    if REF is None:  # C restatement: one full serial run (no session API)
        t0 = time.perf_counter()
        a, _ = ORC.sequential(inst, opol)
        sec = time.perf_counter() - t0
        return dict(value=T / sec, unit="steps/s", cores=1, kind="port",
                    sample=f"C restatement sequential over all {T} orders ({sec:.2f} s, 1 core)",
                    segments_equal=bool(np.array_equal(a, actions)))
    sess = REF.session(inst, opol)
    # size the stretches from a short probe at the head
    probe = min(T, 20_000)
    _, sp = sess.run(probe)
    rate = probe / max(sp, 1e-6)
    n = int(min(T // segments, max(1000, budget_s * rate / segments)))
    total_n, total_s, equal = 0, 0.0, True
    for k in range(segments):
        t0 = k * (T // segments)
        cap, inv = state_at(inst, actions, t0)
        sess.set_state(t0, cap, inv)
        a, sec = sess.run(t0 + n)
        equal &= bool(np.array_equal(a, actions[t0:t0 + n]))
        total_n += n
        total_s += sec
    sess.close()
    return dict(value=total_n / total_s, unit="steps/s", cores=1, kind="reference",
                sample=f"sequential_simulate on {segments} stretches of {n} orders at t = k*T/{segments} "
                       f"({total_n} of {T} orders, {total_s:.2f} s, 1 core), each from the trajectory's exact "
                       f"state there", segments_equal=equal)


def cpu_picard(inst, pol, owner, M, budget_s: float = 15.0):
    """The reference's picard_simulate (threads = every host core) to
    convergence on a prefix of the same instance under the same plan
    (restricted to the prefix), policy horizon T. Every process replays its
    whole window (engine.hpp:313-336), so the full-size run is O(M * T) per
    iteration; the extrapolation to the full horizon scales the sample by the
    first iteration's replay count (sum over processes of last own slot + 1)."""
    from oracle.oracle import REF
    if REF is None:
        return None
    T = int(inst.horizon)
    threads = os.cpu_count() or 1
    opol = oracle_policy_of(pol, T)
    from types import SimpleNamespace as NS

    def prefix(n):
        return NS(nodes=inst.nodes, products=inst.products, horizon=n, product=inst.product[:n], order_t=None,
                  reward_row=inst.reward_row[:n], reward_table=np.asarray(inst.reward_table).ravel(),
                  capacity=inst.capacity, inventory=np.asarray(inst.inventory).ravel())

    def replays(own, n):
        last = np.full(M, -1, np.int64)
        np.maximum.at(last, own[:n], np.arange(n))
        return int((last + 1).sum())

    n, sec, it = 2000, 0.0, 0
    owner = np.asarray(owner, np.int32)
    while True:
        _, it, se, sec = REF.picard_timed(prefix(n), opol, owner[:n], M, 300 * M, threads)
        if sec >= budget_s / 3 or n >= T:
            break
        n = min(T, int(n * max(2.0, min(8.0, (budget_s / 3) / max(sec, 1e-3)))))
    full_replays, sample_replays = replays(owner, T), replays(owner, n)
    return dict(value=n / sec, unit="steps/s", cores=threads, kind="reference",
                sample=f"picard_simulate(threads={threads}) to convergence on the first {n} of {T} orders under "
                       f"the same plan ({sec:.2f} s, {it} iterations)",
                replays_first_iteration={"sample": sample_replays, "full": full_replays},
                extrapolated_full_s_per_iteration=sec / max(it, 1) * full_replays / max(sample_replays, 1))


def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation on rank 0 only.
    The timed K steps are K consecutive stretches of one serial trajectory
    (sequential_simulate over [kT/K, (k+1)T/K) from the carried state), so
    they cover the whole horizon exactly once; each warm-up step runs a short
    head stretch and restores the initial state."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    inst, pol, lib, kind = ref_workload(args.workload)
    T = int(inst.horizon)
    K = max(1, args.steps)
    if kind == "reference":
        sess = lib.session(inst, pol)
        for _ in range(args.warmup):
            sess.run(min(T, max(1, T // (8 * K))))
            sess.set_state(0, inst.capacity, inst.inventory)
        secs, parts = [], []
        for k in range(K):
            a, sec = sess.run((k + 1) * T // K)
            secs.append(sec)
            parts.append(a)
        actions = np.concatenate(parts) if parts else np.zeros(0, np.int32)
        sess.close()
        total = sum(secs)
        sample = (f"sequential_simulate over the whole horizon as {K} consecutive stretches of {T // K} orders "
                  f"(state carried between stretches), {total:.2f} s, 1 core")
    else:
        t0 = time.perf_counter()
        actions, _ = lib.sequential(inst, pol)
        total = time.perf_counter() - t0
        secs = [total / K] * K
        sample = f"C restatement sequential over the whole horizon once ({total:.2f} s, 1 core), split into {K} steps"
    value = T / total
    M = WORKLOADS[args.workload][3]
    picard = None
    if kind == "reference" and not args.no_cpu_picard:
        owner = lib.product_partition(inst, M, 1)
        picard = cpu_picard(inst, pol, owner, M)
        if picard:
            picard["plan"] = "make_product_partition(M, seed 1) (the reference's partitioner)"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s",
            "n_gpus": world, "steps": K, "warmup": args.warmup,
            "ms_per_step": 1000.0 * total / K, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args, world),
            "cpu_baseline": {"value": value, "unit": "steps/s", "cores": 1, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "cpu_picard": picard, "trajectory_hash": trajectory_hash(actions),
            "step_seconds": [round(x, 3) for x in secs],
            "note": "the reference has no GPU path; its serial CPU path is its fastest route to the trajectory "
                    "(its CPU Picard path replays every window per process, cpu_picard)"}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--partition", default="window", choices=sorted(PARTITIONS))
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-picard", action="store_true")
    ap.add_argument("--no-alt-window", action="store_true")
    ap.add_argument("--max-steps", type=int, default=None, help="PicardConfig::max_steps (default 300*M)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_2406_01939_b200 as P
    max_steps = default_window(args.workload) if args.max_steps is None else args.max_steps
    inst, pol, plan, w = make_workload(args.workload, args.partition, max_steps)
    T = w["T"]
    cfg = P.PicardConfig(max_steps=max_steps)
    sim = P.Simulator(inst, pol, device=local)
    sim.set_plan(plan)
    if world > 1:
        uid = [P.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        sim.attach_comm(uid[0], rank, world)

    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up (untimed; includes the flush kernel's first launch)
    res = None
    for _ in range(args.warmup):
        flush.zero_()
        res = sim.simulate_resident(cfg)
    # ---- timed: exactly K steps
    timings, walls = [], []
    with ClockSampler(local, enabled=os.environ.get("BENCH_NO_CLOCKS") is None) as clocks:
        barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            flush.zero_()
            tw = time.perf_counter()
            res = sim.simulate_resident(cfg)
            walls.append(1e3 * (time.perf_counter() - tw))
            timings.append(res.timing)
        t1.record()
        barrier()
    # the engine runs on its own stream: CUDA events recorded on that stream
    # bracket each step (pcd_timing.total_ms); the default-stream events above
    # also count the host work between steps (L2 flush launch, Python) and are
    # reported beside it as wall_ms_per_step
    wall_ms = t0.elapsed_time(t1)
    ms = sum(t["total_ms"] for t in timings)
    if world > 1:
        tt = torch.tensor([ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    ms_per_step = ms / args.steps
    value = T / (ms_per_step / 1000.0)
    actions = sim.download_actions()

    # ---- roofline of the dominant kernel (the sweep)
    tm = timings[-1]
    peaks, peak_src = load_peaks()
    F = flops_per_eval(w["J"])
    sweep_ms = tm["sweep_ms"]
    tc = bool(tm["tc_used"])
    mlp_evals = tm["tc_rows"] if tc else tm["total_evals"]
    achieved_tflops = mlp_evals * F / (sweep_ms / 1000.0) / 1e12 if sweep_ms > 0 else 0.0
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    # DRAM traffic of the sweep from the committed ncu --set full capture
    # (NCU_PROFILE: bytes per policy evaluation) x this run's evaluations per
    # launch
    traffic, hbm_view = None, None
    try:
        with open(os.path.join(ROOT, NCU_PROFILE)) as f:
            prof = json.load(f)
        per_launch_evals = mlp_evals / max(1, tm["sweep_launches"])
        traffic = prof["dram_bytes_per_eval"] * per_launch_evals
        gbs = traffic / (sweep_ms / max(1, tm["sweep_launches"]) / 1000.0) / 1e9
        hbm_view = {"achieved_gbs": gbs, "peak_gbs": peaks.get("hbm_gbs"),
                    "frac": gbs / peaks["hbm_gbs"] if peaks.get("hbm_gbs") else None,
                    "source": f"{NCU_PROFILE} (dram bytes / evaluation) x evaluations / launch"}
    except (OSError, KeyError, ValueError):
        pass
    roofline = {"bound": "tensor", "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tflops / peak, "traffic": traffic, "hbm_view": hbm_view,
                "kernel": ("pp::k_sweep_pp (tc_pp.cu: two 64-row halves per SM, tcgen05.mma kind::f16 M=64 "
                           "fp16x3 split, TMEM accumulators; FP64 exact re-evaluation of rows with margin "
                           "< guard)") if tc else "k_sweep_product<kDual> (FP64 SIMT, exact op order)",
                "per_launch": {"launches": tm["sweep_launches"], "avg_ms": sweep_ms / max(1, tm["sweep_launches"]),
                               "flops_per_eval": F, "mlp_evals": mlp_evals,
                               "algorithmic_flops_per_launch": mlp_evals * F / max(1, tm["sweep_launches"]),
                               "critical_steps": tm["steps_critical"],
                               "us_per_critical_step": 1000.0 * sweep_ms / max(1, tm["steps_critical"])},
                "tc_guard": {"guard": tm["tc_guard"], "derived_score_bound_B": tm["tc_score_bound"],
                             "rows": tm["tc_rows"], "flagged_exact_recheck": tm["tc_flagged"],
                             "fp16x3_wrong_when_flagged": tm["tc_disagree"], "tiles": tm["tc_tiles"]},
                "peak_source": f"{peak_src} bf16_tflops_sustained (MEASURED_PEAKS.json; fp16 dense = bf16)",
                "note": "algorithmic FLOPs = MLP evaluations x (512J+8320); the fp16x3 split issues 3x "
                        "these MACs. Neither roofline binds: each SM runs two 64-row pipelines of dependent "
                        "policy steps (feature build -> 3 MMAs -> argmax -> FP64 re-evaluation of rows "
                        "within the guard) whose latency chains, not tensor or HBM throughput, set the step "
                        "time (see NCU_PROFILE)"}

    # ---- the same trajectory with the CLI-default window (300*M), device-timed
    alt = None
    if max_steps != 300 * w["M"] and not args.no_alt_window:
        acfg = P.PicardConfig(max_steps=300 * w["M"])
        sim.simulate_resident(acfg)
        ams = []
        for _ in range(2):
            flush.zero_()
            ra = sim.simulate_resident(acfg)
            ams.append(ra.timing["total_ms"])
        if world > 1:
            tt = torch.tensor([min(ams)], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ams = [float(tt.item())]
        alt_actions = sim.download_actions()
        alt = {"max_steps": 300 * w["M"], "ms_per_step": min(ams), "value": T / (min(ams) / 1000.0),
               "iterations": ra.iterations_to_converged, "total_evals": ra.total_policy_evals,
               "steps_critical": ra.timing["steps_critical"],
               "same_trajectory": bool(np.array_equal(alt_actions, actions))}

    # ---- the same trajectory with the round-1 calibrated guard (5e-5, no
    # a-priori certificate; verify-mode evidence only), device-timed
    calib = None
    if tc and not args.no_alt_window:
        ccfg = P.PicardConfig(max_steps=max_steps, tc_guard=5e-5)
        sim.simulate_resident(ccfg)
        cms = []
        for _ in range(2):
            flush.zero_()
            rc_ = sim.simulate_resident(ccfg)
            cms.append(rc_.timing["total_ms"])
        if world > 1:
            tt = torch.tensor([min(cms)], device="cuda")
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            cms = [float(tt.item())]
        calib = {"tc_guard": 5e-5, "ms_per_step": min(cms), "value": T / (min(cms) / 1000.0),
                 "flagged_exact_recheck": rc_.timing["tc_flagged"],
                 "same_trajectory": bool(np.array_equal(sim.download_actions(), actions)),
                 "note": "calibrated guard of round 1: exact on every verify-mode run, but without the a-priori "
                         "certificate the default derived guard gives"}

    # ---- e2e through the public one-shot API from pinned host memory
    e2e = None
    if world == 1 and args.e2e_steps > 0:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        pinst = P.Instance(inst.nodes, inst.products, inst.horizon, pin(inst.product), pin(inst.reward_row),
                           pin(inst.reward_table), pin(inst.capacity), pin(inst.inventory))
        pplan = P.PartitionPlan(plan.processes, pin(plan.owner))
        # warm-up: two results alive at once (as in the timed loop) so the
        # library's page-locked result pool holds both buffers
        w1 = P.picard_simulate(pinst, pol, pplan, cfg)
        w2 = P.picard_simulate(pinst, pol, pplan, cfg)
        del w1, w2
        torch.cuda.synchronize()
        t_e = time.perf_counter()
        for _ in range(args.e2e_steps):
            r = P.picard_simulate(pinst, pol, pplan, cfg)
        e2e_s = (time.perf_counter() - t_e) / args.e2e_steps
        assert np.array_equal(r.actions, actions)
        h2d = sum(a.nbytes for a in (inst.product, inst.reward_row, inst.reward_table, inst.capacity,
                                     inst.inventory, plan.owner, pol.w1, pol.b1, pol.w2, pol.b2, pol.w3, pol.b3))
        e2e = {"value": T / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(actions.nbytes), "seconds_per_step": e2e_s,
               "api": "paper_2406_01939_b200.picard_simulate (pcd_picard_simulate: upload, plan CSR, "
                      "fixed point, download)"}

    # ---- CPU baselines (rank 0, N=1): the reference's serial path on a
    # stratified sample, its Picard path on a prefix
    cpu, cpic = None, None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(inst, pol, actions)
        if not args.no_cpu_picard:
            cpic = cpu_picard(inst, pol, plan.owner, plan.processes)

    if rank == 0:
        config = workload_config(args, world)
        line = {"metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
                "config": config,
                "iterations": res.iterations_to_converged,
                "steps_critical": tm["steps_critical"], "total_evals": tm["total_evals"],
                "us_per_critical_step": 1000.0 * ms_per_step / max(1, tm["steps_critical"]),
                "phase_ms": {**{k: tm[k] for k in ("sweep_ms", "prep_ms", "publish_ms", "advance_ms")},
                             "engine_total_ms": tm["total_ms"],
                             "host_wall_ms_per_step": [round(w, 2) for w in walls],
                             "wall_ms_per_step": wall_ms / args.steps,
                             "host_gap_ms": tm["total_ms"] - sum(tm[k] for k in ("sweep_ms", "prep_ms", "publish_ms",
                                                                                    "advance_ms"))},
                "roofline": roofline, "cpu_baseline": cpu, "cpu_picard": cpic, "e2e": e2e,
                "cli_default_window": alt, "calibrated_guard": calib,
                "trajectory_hash": trajectory_hash(actions),
                "gpu_launches": int(sum(t["kernel_launches"] for t in timings)),
                "clocks": clocks.summary()}
        if cpu:
            line["speedup_vs_cpu_serial"] = value / cpu["value"]
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    sim.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
