timeout 600 python -m pytest tests/test_wire.py -x -q > gpurun_out/pytest_wire.log 2>&1; echo wire=$?
tail -2 gpurun_out/pytest_wire.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'])"
