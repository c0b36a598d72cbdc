timeout 600 python -m pytest tests/test_gpu_stream.py -x -q > gpurun_out/pytest_stream.log 2>&1; echo stream=$?
tail -2 gpurun_out/pytest_stream.log
CS_FUSED=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cycle_reduce_v2|k_scan_warp|k_bounds_tile" -s 3 -c 3 -o gpurun_out/leg2 python tools/tools_fused_one.py > gpurun_out/leg_ncu.log 2>&1; echo ncu=$?
tail -2 gpurun_out/leg_ncu.log
