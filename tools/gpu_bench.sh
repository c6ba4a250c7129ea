cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --cpu-steps 1 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -3 gpurun_out/bench.err
