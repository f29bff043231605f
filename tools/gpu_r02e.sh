mkdir -p gpurun_out/r02e
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_kernels.py -q -x -s -k "derived_guard or tensor_core or guard_scales or tc" > gpurun_out/r02e/tc_tests.log 2>&1
timeout 600 python tools/guard_time.py 500000 0 5e-5 > gpurun_out/r02e/guard_time.log 2>&1
tail -12 gpurun_out/r02e/tc_tests.log; cat gpurun_out/r02e/guard_time.log
