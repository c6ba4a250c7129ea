# config 4 (stream with growth) and config 5 (8-view batch) measurements
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2; grep -E "^(FAILED|ERROR)" gpurun_out/pytest_gpu.log | head
timeout 300 python bench.py --steps 30 --no-cpu-baseline > gpurun_out/bench_q.json 2> gpurun_out/bench_q.err; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_q.json'));print('cfg3', d['value'], d['e2e']['value'])"
timeout 300 python tools/stream_bench.py --teacher 200000 --frames 100 > gpurun_out/stream_small.json 2> gpurun_out/stream_small.err; echo stream_small rc=$?
tail -3 gpurun_out/stream_small.err; cat gpurun_out/stream_small.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --batched --config 5 --steps 5 --warmup 3 > gpurun_out/batched_c5.json 2> gpurun_out/batched_c5.err; echo c5 rc=$?
tail -3 gpurun_out/batched_c5.err; cat gpurun_out/batched_c5.json
timeout 900 python tools/stream_bench.py > gpurun_out/stream_full.json 2> gpurun_out/stream_full.err; echo stream_full rc=$?
tail -3 gpurun_out/stream_full.err; cat gpurun_out/stream_full.json
