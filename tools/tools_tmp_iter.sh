timeout 900 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/s51_c3.log 2>&1
for i in 1 2; do timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/s51_c5.log 2>&1; tail -1 gpurun_out/s51_c5.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['latency_ms'], d['device_ms_per_slice_median'], d['alerts'])"; done
timeout 600 python bench.py --workload c1 > gpurun_out/s51_c1.log 2>&1
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/s51_c5.log 2>&1; tail -1 gpurun_out/s51_c5.log | python -c "import json,sys; d=json.load(sys.stdin); print(d['latency_ms'], d['device_ms_per_slice_median'], d['alerts'])"
