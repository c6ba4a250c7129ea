cd $GRAFT_REPO_ROOT
timeout 300 python tools/bin_bench.py > gpurun_out/binbench.log 2>&1; echo rc=$?; tail -2 gpurun_out/binbench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bin_launches.csv python tools/bin_bench.py --iters 3 > gpurun_out/bin_ncu.log 2>&1; echo ncu rc=$?
