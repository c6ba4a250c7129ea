# round evidence: tests, smoke, full bench (+ CPU baseline), reference arm,
# clean per-step launch list, one ncu --set full capture of the step's kernels
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed" gpurun_out/pytest_gpu.log | tail -2
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?; cat gpurun_out/bench_ref.json
timeout 300 python tools/step_launches.py > gpurun_out/sl_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/step_launches.py > gpurun_out/sl_ncu.log 2>&1; echo launches rc=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"blend_bwd|blend_fwd|adam_apply|chain_grad|chain_flags|count_hist|place_kernel|Onesweep|ssim|loss_grad|preprocess_fwd" -c 14 -o gpurun_out/prof_r1 python tools/step_launches.py 1 > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
