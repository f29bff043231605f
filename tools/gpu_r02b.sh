set -x
mkdir -p gpurun_out/r02b
./tools/mma_accum_probe > gpurun_out/r02b/mma_probe.log 2>&1
timeout 600 python -m pytest tests/test_linear.py -q -m gpu > gpurun_out/r02b/linear_tests.log 2>&1
timeout 600 python tools/c4_mlp.py > gpurun_out/r02b/c4_mlp.jsonl 2> gpurun_out/r02b/c4_mlp.err
tail -3 gpurun_out/r02b/linear_tests.log
