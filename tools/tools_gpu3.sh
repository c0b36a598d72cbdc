timeout 600 python -m pytest tests/test_gpu_stream.py -q > gpurun_out/pytest_stream.log 2>&1; echo stream=$?
tail -3 gpurun_out/pytest_stream.log
