# round-end evidence, part 2: one ncu --set full capture of the step's kernels
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"blend_bwd|blend_fwd|adam_apply|chain_grad|count_hist|place_kernel|Onesweep|ssim|loss_grad|preprocess_fwd" -s 30 -c 12 -o gpurun_out/prof_r1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
