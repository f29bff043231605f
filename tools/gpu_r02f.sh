mkdir -p gpurun_out/r02f
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02f/gputests.log 2>&1
tail -3 gpurun_out/r02f/gputests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02f/bench.json 2> gpurun_out/r02f/bench.err
tail -c 600 gpurun_out/r02f/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cpu-picard --e2e-steps 0 --no-alt-window > gpurun_out/r02f/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_pp -s 20 -c 1 -o gpurun_out/r02f/sweep_pp python tools/tc_ncu_target.py 100 10000 10000000 65536 --chunk --window 500000 --cap 22 > gpurun_out/r02f/ncu_full.log 2>&1
ls gpurun_out/r02f
