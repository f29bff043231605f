set -x
mkdir -p gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "derived_guard or tensor_core or guard_scales" -s > gpurun_out/r02d/tc_tests.log 2>&1
timeout 600 python tools/guard_time.py 500000 0 5e-5 1e-3 > gpurun_out/r02d/guard_time.log 2>&1
tail -5 gpurun_out/r02d/tc_tests.log; cat gpurun_out/r02d/guard_time.log
