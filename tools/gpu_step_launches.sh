cd $GRAFT_REPO_ROOT
timeout 300 python tools/step_launches.py > gpurun_out/sl_plain.log 2>&1; echo plain rc=$?; cat gpurun_out/sl_plain.log | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/step_launches.py > gpurun_out/sl_ncu.log 2>&1; echo ncu rc=$?
