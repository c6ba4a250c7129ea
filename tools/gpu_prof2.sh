cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"blend_bwd|chain_adam" -s 2 -c 2 -o gpurun_out/prof_r1b python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_full.log
