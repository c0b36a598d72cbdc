# Round evidence (refresh): smoke, full GPU suite, benches (ours c2/c3/c5 +
# reference arm + fit + ingest), ncu launch list and one full capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/bench_c5.log 2>&1; echo c5=$?
timeout 600 python bench.py --workload c1 > gpurun_out/bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --workload c1 --impl reference --steps 3 --warmup 3 > gpurun_out/bench_c1_ref.log 2>&1; echo c1ref=$?
timeout 600 python bench.py --c2-split halo --steps 5 > gpurun_out/bench_c2_halo.log 2>&1; echo halo=$?
timeout 1200 python tools/tools_halo_bench.py > gpurun_out/halo_bench.log 2>&1; echo halo_bench=$?
timeout 900 python tools/tools_suite_bench.py > gpurun_out/suite.log 2>&1; echo suite=$?
timeout 600 python tools/tools_fit_bench.py 1024 > gpurun_out/fit_bench.log 2>&1; echo fit=$?
timeout 600 python tools/tools_ingest_bench.py > gpurun_out/ingest.log 2>&1; echo ingest=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo ncu1=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_cycle_reduce_v2|k_scan_warp|k_score_lut|k_bounds_tile|k_detect_flags|k_wire_expand" -s 8 -c 7 -o gpurun_out/full python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/b_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; for f in bench bench_ref bench_c3 bench_c5; do tail -1 gpurun_out/$f.log | cut -c1-300; done
