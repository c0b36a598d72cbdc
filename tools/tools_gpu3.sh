timeout 600 python tools/tools_variants.py 3700000 0,1 > gpurun_out/variants.log 2>&1; echo var=$?
cat gpurun_out/variants.log
