# compute-sanitizer memcheck over the GPU test suite minus the full-scale cases
mkdir -p gpurun_out
timeout 5000 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 --print-limit 20 \
  python -m pytest tests -m gpu -q -p no:cacheprovider -x \
  -k "not full and not scale and not c1_scale and not 100k and not suite and not fit_1024" > gpurun_out/r2_memcheck_suite.log 2>&1
echo memcheck_suite=$?
tail -5 gpurun_out/r2_memcheck_suite.log
grep -c "Invalid\|ERROR SUMMARY" gpurun_out/r2_memcheck_suite.log
