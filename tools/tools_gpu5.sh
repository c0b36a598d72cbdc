# Device GBDT fit: parity tests, then the batch benchmark.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fit.py -x -q > gpurun_out/pytest_fit.log 2>&1; echo fit_tests=$?
timeout 600 python tools/tools_fit_bench.py 1024 > gpurun_out/fit_bench.log 2>&1; echo fit_bench=$?
tail -25 gpurun_out/pytest_fit.log; tail -3 gpurun_out/fit_bench.log
