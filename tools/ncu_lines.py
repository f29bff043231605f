"""Per-source-line hot spots of one ncu capture (compile with -lineinfo):
warp-stall samples and executed warp instructions of every CUDA line.

  python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out = "?", None, []
for r in csv.reader(io.StringIO(raw)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or r[0] == "Function Name":
        continue
    try:
        s = int(r[4] or 0)
        n = int(r[7] or 0)
    except (ValueError, IndexError):
        continue
    if s or n:
        out.append((s, n, f"{cur}:{r[0]}", r[1].strip()[:100]))
tot_s = sum(o[0] for o in out) or 1
tot_n = sum(o[1] for o in out) or 1
print(f"total stall samples {tot_s}, warp instructions {tot_n}")
for s, n, line, src in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*n/tot_n:5.1f}% ins  {line:<22} {src}")
