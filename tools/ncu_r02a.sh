set -x
mkdir -p gpurun_out/r02a
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cpu-picard --e2e-steps 0 --no-alt-window > gpurun_out/r02a/bench_under_ncu.log 2>&1
timeout 300 python tools/tc_ncu_target.py 100 10000 10000000 65536 --chunk --window 500000 --evals 21 > gpurun_out/r02a/evals21.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_pp -s 20 -c 1 -o gpurun_out/r02a/sweep_pp python tools/tc_ncu_target.py 100 10000 10000000 65536 --chunk --window 500000 --cap 22 > gpurun_out/r02a/ncu_full.log 2>&1
ls -la gpurun_out/r02a
