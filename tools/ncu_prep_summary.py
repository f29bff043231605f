"""Summarise an ncu capture of the cache / dynamics kernels (prep + checkpoint
advance) into profiles/ JSON: per kernel the duration, DRAM bytes, achieved
HBM GB/s against the measured peak (MEASURED_PEAKS.json), L2 hit rate.

  python tools/ncu_prep_summary.py REPORT.ncu-rep OUT.json "capture command"
"""
import csv
import io
import json
import subprocess
import sys

rep, out_path, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
try:
    peak = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs")
except OSError:
    peak = 6650.0
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "Tbyte": 1e12}
tscale = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1.0}
out = []
for v in rows[2:]:
    g = lambda n: v[h.index(n)] if n in h else None
    name = g("Kernel Name").split("(")[0]
    t = float(g("gpu__time_duration.sum").replace(",", "")) * tscale[u[h.index("gpu__time_duration.sum")]]
    rd = float(g("dram__bytes_read.sum").replace(",", "")) * scale[u[h.index("dram__bytes_read.sum")]]
    wr = float(g("dram__bytes_write.sum").replace(",", "")) * scale[u[h.index("dram__bytes_write.sum")]]
    gbs = (rd + wr) / t / 1e9 if t > 0 else 0.0
    out.append({"kernel": name, "us": t * 1e6, "dram_read_bytes": rd, "dram_write_bytes": wr,
                "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak if peak else None,
                "l2_hit_pct": float(g("lts__t_sector_hit_rate.pct") or 0),
                "grid": g("launch__grid_size"), "block": g("launch__block_size"),
                "issue_active_pct": float(g("smsp__issue_active.avg.pct_of_peak_sustained_active") or 0)})
json.dump({"capture": cmd, "peak_source": "MEASURED_PEAKS.json hbm_gbs", "kernels": out}, open(out_path, "w"), indent=1)
for k in out:
    print(f"{k['kernel'][:40]:40s} {k['us']:8.1f} us {k['achieved_gbs']:8.1f} GB/s ({100 * (k['frac'] or 0):.1f}%) "
          f"L2 hit {k['l2_hit_pct']:.0f}%")
