for pf in 0 1 2; do
  echo "pf=$pf"; PCD_TC_PF=$pf python bench.py --steps 2 --warmup 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['phase_ms'])"
  PCD_TC_PF=$pf PCD_TC_PROF=1 python tests/tc_ncu_target.py 100 10000 10000000 65536 product --cap 2>&1 | grep tcprof | tail -2
done
