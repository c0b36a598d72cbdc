timeout 900 python bench.py --workload c5 --steps 50 --warmup 5 > gpurun_out/bench_c5.log 2>&1; echo c5=$?
tail -1 gpurun_out/bench_c5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['latency_ms'], d['device_phase_ms_last_slice'])"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -2 gpurun_out/pytest_gpu.log
