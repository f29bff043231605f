#!/bin/bash
# A/B of prebuilt engine variants (ab/<name>.so) on the C3 fixed point at the bench window:
#   bash tools/ab_guard.sh name1 name2 ... -> "name device_ms" lines (2 rounds)
L=paper_2406_01939_b200/libpicard_b200.so
cp $L ab/_orig.so
for r in 1 2; do
  for v in "$@"; do
    cp ab/$v.so $L
    python tools/guard_time.py 300000 0 2>&1 | grep "guard=" | tail -1 | sed "s/^/$v /"
  done
done
cp ab/_orig.so $L
