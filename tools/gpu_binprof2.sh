cd $GRAFT_REPO_ROOT
timeout 300 python tools/bin_bench.py --iters 3 > gpurun_out/binbench.log 2>&1; echo rc=$?; tail -2 gpurun_out/binbench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"place_kernel" -s 3 -c 1 -o gpurun_out/prof_bin2 python tools/bin_bench.py --iters 2 > gpurun_out/ncu_bin.log 2>&1; echo ncu rc=$?
