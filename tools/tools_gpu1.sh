# Round evidence: smoke, GPU tests, bench (ours + reference arm), launch list, ncu full capture.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cycle_reduce_v2|k_scan_warp|k_score_lut|k_bounds_tile|k_detect_flags" -s 8 -c 6 -o gpurun_out/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -2; cat gpurun_out/bench.log gpurun_out/bench_ref.log | tail -4
