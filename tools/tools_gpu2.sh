timeout 300 python tools/tools_fused_check.py > gpurun_out/fused_check.log 2>&1; echo check=$?
cat gpurun_out/fused_check.log | head -4
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
