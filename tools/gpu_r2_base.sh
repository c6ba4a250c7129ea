# round 2 baseline: bench (no CPU), then one ncu --set full capture of the
# backward blend, forward blend and placement kernel with atomic counters
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err; echo bench rc=$?
timeout 300 python tools/step_launches.py 1 > gpurun_out/r2_sl_plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,l1tex__t_set_accesses_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,lts__t_requests_op_red.sum \
  -k regex:"blend_bwd|blend_fwd|place_kernel|count_hist" -c 4 -o gpurun_out/r2_base python tools/step_launches.py 1 > gpurun_out/r2_ncu.log 2>&1; echo ncu rc=$?
