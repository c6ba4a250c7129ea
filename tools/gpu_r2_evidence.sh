# round-2 evidence: per-step launch list (time + DRAM bytes, cold cache as ncu
# serialises), then one ncu --set full capture of the step's kernels with the
# L2 atomic/reduction counters (the north star's atomic-throughput evidence)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/step_launches.py 3 > gpurun_out/ev_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv python tools/step_launches.py 3 > gpurun_out/ev_ncu1.log 2>&1; echo launches rc=$?
timeout 1200 ncu --profile-from-start off --set full --import-source on --clock-control none \
  --metrics lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_requests_op_red.sum,lts__t_requests_op_atom.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum \
  -k regex:"blend_bwd|blend_fwd|place_kernel|count_hist|adam_list|adam_apply|gather_short|gather_long|ssim_stats|ssim_adjoint|loss_grad|loss_tail|preprocess_fwd|chain_grad|chain_flags|Onesweep" -c 20 -o gpurun_out/r2_full python tools/step_launches.py 1 > gpurun_out/ev_ncu2.log 2>&1; echo full rc=$?
