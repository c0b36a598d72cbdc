# Wire v2 + ingest check: GPU tests, bench (c2), ingest bench.
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python tools/tools_ingest_bench.py > gpurun_out/ingest.log 2>&1; echo ingest=$?
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/bench.log; tail -3 gpurun_out/ingest.log
