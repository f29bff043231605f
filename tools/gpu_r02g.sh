mkdir -p gpurun_out/r02g
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc_kernels.py tests/test_gpu_fullscale.py -q -x -k "derived_guard or tensor_core or guard_scales or tc or verify" > gpurun_out/r02g/tc_tests.log 2>&1
tail -3 gpurun_out/r02g/tc_tests.log
timeout 600 python tools/guard_time.py 500000 0 5e-5 > gpurun_out/r02g/guard_time.log 2>&1; cat gpurun_out/r02g/guard_time.log
python tools/phase_profile_c3.py 500000 0 40 2> gpurun_out/r02g/phase_derived.log
