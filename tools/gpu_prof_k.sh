# usage: bash tools/gpu_prof_k.sh <kernel regex> <report name>
cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$1" -s 3 -c 1 -o gpurun_out/$2 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_$2.log 2>&1; echo ncu rc=$?
