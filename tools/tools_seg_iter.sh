# Single-read segmentation iteration on the box: fused-path parity subset,
# full-scale fused-vs-two-pass bit check with timings, one ncu capture.
# Usage: bash tools/tools_seg_iter.sh TAG
T=${1:-seg}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "fused or single-read or golden or c1_scale" > gpurun_out/${T}_pytest.log 2>&1; echo pytest=$?
timeout 400 python tools/tools_fused_check.py > gpurun_out/${T}_fused_check.log 2>&1; echo fc=$?
CS_BENCH_FUSED=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_segment_range" -s 1 -c 1 -o gpurun_out/${T}_seg python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/${T}_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/${T}_pytest.log; tail -12 gpurun_out/${T}_fused_check.log
