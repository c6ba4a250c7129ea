# per-change gate: GPU tests, smoke, one short bench line (no CPU baseline)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'fps', d['render_fps']); print(d['roofline']['kernel_ms'])"
