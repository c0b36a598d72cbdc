set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rca.py tests/test_gpu_fit.py -x -q > gpurun_out/pytest_rca.log 2>&1; echo rca_tests=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
tail -25 gpurun_out/pytest_rca.log; tail -1 gpurun_out/bench.log | cut -c1-600
