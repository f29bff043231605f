# final measurement set of a round: GPU tests, bench (C3 + C2), reference arm,
# launch list, ncu of the sweep / cache kernels / verification kernel, smoke
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s > gpurun_out/final/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/final/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-picard > gpurun_out/final/bench_c2.json 2> gpurun_out/final/bench_c2.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cpu-picard --e2e-steps 0 --no-alt-window > gpurun_out/final/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_pp -s 30 -c 1 -o gpurun_out/final/sweep_pp python tools/tc_ncu_target.py 100 10000 10000000 65536 --wplan --window 350000 --cap 32 > gpurun_out/final/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_effective|k_xinit|k_hist_prefix|k_advance|k_tau|k_seg_count|k_window_load" -s 180 -c 7 -o gpurun_out/final/prep python tools/tc_ncu_target.py 100 10000 10000000 65536 --wplan --window 350000 --cap 40 > gpurun_out/final/ncu_prep.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spec_verify -s 40 -c 1 -o gpurun_out/final/spec_verify python tools/tc_ncu_target.py 100 10000 10000000 65536 --wplan --window 350000 --cap 45 > gpurun_out/final/ncu_spec.log 2>&1
timeout 300 python tools/tc_ncu_target.py 100 10000 10000000 65536 --wplan --window 350000 --evals 31 > gpurun_out/final/evals31.log 2>&1
grep -E "passed|failed|rc=" gpurun_out/final/gpu_tests.log | tail -2; tail -c 250 gpurun_out/final/bench.json; cat gpurun_out/final/smoke.log
