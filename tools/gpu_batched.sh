cd $GRAFT_REPO_ROOT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --batched --steps 10 --warmup 2 > gpurun_out/batched.json 2> gpurun_out/batched.err; echo rc=$?
tail -5 gpurun_out/batched.err; cat gpurun_out/batched.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; echo ref rc=$?; tail -2 gpurun_out/ref.err; cat gpurun_out/ref.json
