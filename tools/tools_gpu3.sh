timeout 300 python tools/tools_fused_check.py > gpurun_out/fused_check.log 2>&1; echo check=$?
head -4 gpurun_out/fused_check.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python tools/tools_launches_run.py > /dev/null 2>&1
