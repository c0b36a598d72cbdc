set -x
mkdir -p gpurun_out
timeout 300 python tools/tools_sanitize.py > gpurun_out/r2_sanitize_plain.log 2>&1; echo plain=$?
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python tools/tools_sanitize.py > gpurun_out/r2_sanitize_memcheck.log 2>&1; echo memcheck=$?
timeout 1200 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/tools_sanitize.py > gpurun_out/r2_sanitize_racecheck.log 2>&1; echo racecheck=$?
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/tools_sanitize.py > gpurun_out/r2_sanitize_synccheck.log 2>&1; echo synccheck=$?
timeout 600 ncu --nvtx --print-summary per-nvtx --metrics gpu__time_duration.sum -c 60 python tools/tools_sanitize.py > gpurun_out/r2_nvtx.log 2>&1; echo nvtx=$?
for f in plain memcheck racecheck synccheck; do echo "== $f"; tail -4 gpurun_out/r2_sanitize_$f.log; done; grep -c "cs_run" gpurun_out/r2_nvtx.log
