cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"adam_apply|chain_grad" -s 4 -c 2 -o gpurun_out/prof_r1g python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
