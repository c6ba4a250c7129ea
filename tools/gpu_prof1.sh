cd $GRAFT_REPO_ROOT
timeout 300 python tools/diag_slim.py > gpurun_out/diag_slim.log 2>&1; echo diag rc=$?
cat gpurun_out/diag_slim.log
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"blend_bwd|chain_adam|blend_fwd|count_kernel|emit_kernel" -s 5 -c 5 -o gpurun_out/prof_r1a python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out
