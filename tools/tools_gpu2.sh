timeout 300 python tools/tools_fused_check.py > gpurun_out/fused_check.log 2>&1; echo check=$?
cat gpurun_out/fused_check.log
timeout 300 python tools/tools_fused_ablation.py > gpurun_out/ablation.log 2>&1; echo abl=$?
cat gpurun_out/ablation.log
timeout 600 python -m pytest tests -m gpu -x -q -k "fused" > gpurun_out/pytest_fused.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_fused.log
