"""Summarise one ncu --set full capture of the sweep kernel into profiles/ JSON.

  python tools/ncu_summary.py REPORT.ncu-rep OUT.json "capture command" evals_in_launch
"""
import csv
import io
import json
import subprocess
import sys

rep, out_path, cmd, evals = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__m_xbar2l1tex_read_sectors_mem_lg_op_ld.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__func_cache_config"]
metrics = {}
for n in want:
    if n in h:
        try:
            metrics[n] = {"unit": u[h.index(n)], "value": float(v[h.index(n)].replace(",", ""))}
        except ValueError:
            metrics[n] = {"unit": u[h.index(n)], "value": v[h.index(n)]}
stalls = {}
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled_") and "not_issued" not in n:
        try:
            x = int(float(v[i]))
        except ValueError:
            continue
        if x > 0:
            stalls[n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = x
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
rd, wr = metrics["dram__bytes_read.sum"], metrics["dram__bytes_write.sum"]
traffic = rd["value"] * scale[rd["unit"]] + wr["value"] * scale[wr["unit"]]
summary = {"capture": cmd, "evals_in_launch": evals, "dram_bytes_per_launch": traffic,
           "dram_bytes_per_eval": traffic / evals, "metrics": metrics,
           "stall_samples": dict(sorted(stalls.items(), key=lambda kv: -kv[1]))}
json.dump(summary, open(out_path, "w"), indent=1)
print(json.dumps(summary)[:800])
