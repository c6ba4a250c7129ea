# usage: bash tools/gpu_sanitize.sh <memcheck|racecheck|synccheck>  (one tool per gpurun call)
cd $GRAFT_REPO_ROOT
timeout 300 python tools/sanitize_smoke.py > gpurun_out/san_plain.log 2>&1; echo plain rc=$?
timeout 1500 compute-sanitizer --tool $1 --error-exitcode 99 --print-limit 50 python tools/sanitize_smoke.py > gpurun_out/san_$1.log 2>&1; echo $1 rc=$?
tail -5 gpurun_out/san_$1.log
