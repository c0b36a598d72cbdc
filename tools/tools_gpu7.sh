set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fit.py -x -q > gpurun_out/pytest_fit.log 2>&1; echo fit_tests=$?
CS_FIT_PROFILE=1 timeout 300 python tools/tools_fit_one.py 1 50 > gpurun_out/fit_prof.log 2>&1
for M in 148 296; do timeout 300 python tools/tools_fit_one.py $M 50; done > gpurun_out/fit_sweep.log 2>&1
timeout 600 python tools/tools_fit_bench.py 1024 > gpurun_out/fit_bench.log 2>&1; echo fit_bench=$?
tail -3 gpurun_out/pytest_fit.log; cat gpurun_out/fit_prof.log gpurun_out/fit_sweep.log; tail -1 gpurun_out/fit_bench.log
