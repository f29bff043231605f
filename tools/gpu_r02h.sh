mkdir -p gpurun_out/r02h
timeout 900 python tools/window_sweep.py 200000 300000 500000 1000000 > gpurun_out/r02h/ws_65536.jsonl 2>&1
WS_M=32768 timeout 600 python tools/window_sweep.py 300000 500000 1000000 > gpurun_out/r02h/ws_32768.jsonl 2>&1
WS_M=16384 timeout 600 python tools/window_sweep.py 500000 1000000 > gpurun_out/r02h/ws_16384.jsonl 2>&1
timeout 600 python bench.py --workload c2 --steps 5 --warmup 3 --no-cpu-picard > gpurun_out/r02h/bench_c2.json 2> gpurun_out/r02h/bench_c2.err
cat gpurun_out/r02h/*.jsonl
