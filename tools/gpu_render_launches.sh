cd $GRAFT_REPO_ROOT
SB_RENDER=1 timeout 300 python tools/step_launches.py 3 > /dev/null 2>&1 && \
SB_RENDER=1 timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/render_warm.csv python tools/step_launches.py 3 > /dev/null 2>&1; echo rc=$?
