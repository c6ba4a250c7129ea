# config-5 batched step at world 1 with each exchange (the packed one reports its wire rows)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
for ex in packed packed_sharded sharded allreduce; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29521 bench.py --batched --config 5 --exchange $ex --steps 5 --warmup 3 > gpurun_out/c5_$ex.json 2> gpurun_out/c5_$ex.err; echo $ex rc=$?
  grep '^{' gpurun_out/c5_$ex.json | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['config']['exchange_rows'], d['config']['reached_rows_this_rank'])"
done
