# per-change gate: GPU tests, a short config-3 bench, the config-5 batched bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print('cfg3', d['value'], d['e2e']['value'], d['invalid_timed_runs'], d['roofline']['kernel_ms'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --batched --config 5 --steps 5 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo c5 rc=$?
grep '^{' gpurun_out/c5.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print('c5', d['value'], d['ms_per_step'], d['e2e']['value'])"
