timeout 600 python tools/tools_variants.py 3700000 0 > gpurun_out/variants.log 2>&1; echo var=$?
cat gpurun_out/variants.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
