# GPU tests, then the batched step at world 1: config 3 (one view) and config 5 (8 views)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
for c in 3 5; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2954$c bench.py --batched --config $c --steps 20 --warmup 3 > gpurun_out/bq_c$c.json 2> gpurun_out/bq_c$c.err; echo c$c rc=$?
  grep '^{' gpurun_out/bq_c$c.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['e2e']['value'])"
done
