mkdir -p gpurun_out/r02k
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02k/bench.json 2> gpurun_out/r02k/bench.err
tail -c 400 gpurun_out/r02k/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02k/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-cpu-picard --e2e-steps 0 --no-alt-window > gpurun_out/r02k/bench_under_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_pp -s 30 -c 1 -o gpurun_out/r02k/sweep_pp python tools/tc_ncu_target.py 100 10000 10000000 65536 --chunk --window 300000 --cap 32 > gpurun_out/r02k/ncu_full.log 2>&1
timeout 300 python tools/tc_ncu_target.py 100 10000 10000000 65536 --chunk --window 300000 --evals 31 > gpurun_out/r02k/evals31.log 2>&1
cat gpurun_out/r02k/evals31.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02k/smoke.log 2>&1; cat gpurun_out/r02k/smoke.log
