# usage: bash tools/gpu_prof_k2.sh <kernel regex> <report name> : one ncu --set full capture of the step's kernels
cd $GRAFT_REPO_ROOT
timeout 300 python tools/step_launches.py 1 > gpurun_out/k_plain.log 2>&1 && \
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:"$1" -o gpurun_out/$2 python tools/step_launches.py 1 > gpurun_out/k_ncu.log 2>&1; echo ncu rc=$?
