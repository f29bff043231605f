mkdir -p gpurun_out/r02l
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02l/gputests.log 2>&1
tail -3 gpurun_out/r02l/gputests.log
python tools/guard_time.py 300000 0 5e-5 2>&1
python tools/phase_profile_c3.py 300000 0 40 2> gpurun_out/r02l/phase.log
