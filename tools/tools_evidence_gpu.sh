# Round evidence (refresh): smoke, full GPU suite, benches (ours c2/c3/c5/c1 +
# reference arms + halo + the two-pass path), heuristic / suite / ingest
# benches, ncu launch list and one full capture.  Outputs gpurun_out/r2_*.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke=$?
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo ref=$?
CS_BENCH_FUSED=0 timeout 900 python bench.py --no-cpu-baseline --no-parity > gpurun_out/r2_bench_twopass.log 2>&1; echo twopass=$?
timeout 900 python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2_bench_c3.log 2>&1; echo c3=$?
timeout 600 python bench.py --workload c5 --no-cpu-baseline > gpurun_out/r2_bench_c5.log 2>&1; echo c5=$?
CS_HOST_PROFILE=1 timeout 600 python bench.py --workload c5 --no-cpu-baseline --steps 6 > gpurun_out/r2_c5_host.log 2>&1; echo c5host=$?
timeout 600 python bench.py --workload c1 > gpurun_out/r2_bench_c1.log 2>&1; echo c1=$?
timeout 600 python bench.py --workload c1 --impl reference > gpurun_out/r2_bench_c1_ref.log 2>&1; echo c1ref=$?
timeout 600 python bench.py --c2-split halo --steps 5 > gpurun_out/r2_bench_c2_halo.log 2>&1; echo halo=$?
CS_STAGE_ITERS=1 timeout 900 python tools/tools_heuristic_bench.py > gpurun_out/r2_heuristic.log 2>&1; echo heur=$?
timeout 900 python tools/tools_suite_bench.py > gpurun_out/r2_suite.log 2>&1; echo suite=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r2_b_ncu.log 2>&1; echo ncu1=$?
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_segment_range|k_score_lut|k_detect_win|k_records_scatter|k_records_count|k_stage_blocks" -s 12 -c 6 -o gpurun_out/r2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/r2_b_full.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/r2_pytest_gpu.log; tail -2 gpurun_out/r2_smoke.log; for f in bench bench_ref bench_twopass bench_c3 bench_c5 bench_c1 heuristic; do tail -1 gpurun_out/r2_$f.log | cut -c1-300; done
