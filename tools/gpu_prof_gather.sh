cd $GRAFT_REPO_ROOT
timeout 300 python tools/step_launches.py 1 > gpurun_out/g_plain.log 2>&1 && \
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/step_launches.py 3 > gpurun_out/sl_ncu_w.log 2>&1; echo warm rc=$?
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"gather|loss_tail" -c 3 -o gpurun_out/r2_gather python tools/step_launches.py 1 > gpurun_out/g_ncu.log 2>&1; echo ncu rc=$?
