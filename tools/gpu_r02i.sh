mkdir -p gpurun_out/r02i
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02i/gputests.log 2>&1
tail -3 gpurun_out/r02i/gputests.log
timeout 600 python tools/window_sweep.py 200000 300000 500000 > gpurun_out/r02i/ws.jsonl 2>&1; cat gpurun_out/r02i/ws.jsonl
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02i/bench.json 2> gpurun_out/r02i/bench.err
tail -c 300 gpurun_out/r02i/bench.json
