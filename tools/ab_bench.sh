#!/bin/bash
# A/B of two prebuilt engine libraries on the same GPU box (build each variant,
# copy it to ab/<name>.so; ab/ is git-ignored but travels with gpurun):
#   bash tools/ab_bench.sh name1 name2 [rounds]  -> "name ms_per_step sweep_ms prep_ms" lines
L=paper_2406_01939_b200/libpicard_b200.so
for r in $(seq ${3:-3}); do
  for v in $1 $2; do
    cp ab/$v.so $L
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('$v', round(d['ms_per_step'],2), round(d['phase_ms']['sweep_ms'],2), round(d['phase_ms']['prep_ms'],2))"
  done
done
