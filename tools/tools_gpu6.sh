# Device fit profile: timing sweep, then one ncu capture with source lines.
set -x
mkdir -p gpurun_out
for M in 1 8 148 296; do timeout 300 python tools/tools_fit_one.py $M 50; done > gpurun_out/fit_sweep.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gbdt_fit -c 1 -o gpurun_out/fit_full python tools/tools_fit_one.py 2 20 > gpurun_out/fit_ncu.log 2>&1; echo ncu=$?
cat gpurun_out/fit_sweep.log; tail -3 gpurun_out/fit_ncu.log
