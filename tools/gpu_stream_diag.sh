cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print('cfg3', d['value'], d['e2e']['value'], d['invalid_timed_runs'])"
timeout 900 python tools/stream_bench.py ${STREAM_ARGS} > gpurun_out/stream_diag.json 2> gpurun_out/stream_diag.err; echo stream rc=$?
tail -3 gpurun_out/stream_diag.err; cat gpurun_out/stream_diag.json
