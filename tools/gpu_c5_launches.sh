# config 5 batched step: timing + ncu launch list (one GPU, world size 1)
cd $GRAFT_REPO_ROOT
RUN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --batched --config 5"
timeout 600 $RUN --steps 5 --warmup 3 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo c5 rc=$?
python -c "import json;d=json.load(open('gpurun_out/c5.json'));print('c5', d['value'], d['ms_per_step'], d['e2e']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv $RUN --steps 1 --warmup 3 > gpurun_out/c5_ncu.log 2>&1; echo ncu rc=$?
timeout 900 python tools/stream_bench.py > gpurun_out/stream_diag.json 2> gpurun_out/stream_diag.err; echo stream rc=$?
tail -3 gpurun_out/stream_diag.err; cat gpurun_out/stream_diag.json
