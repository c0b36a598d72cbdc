CS_FUSED=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cycle_reduce_tpc|k_scan_events|k_bounds" -s 3 -c 3 -o gpurun_out/leg python tools/tools_fused_one.py > gpurun_out/leg_ncu.log 2>&1; echo ncu=$?
tail -3 gpurun_out/leg_ncu.log
