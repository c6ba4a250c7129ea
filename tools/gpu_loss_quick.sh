cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_kats.py tests/test_gpu_fullsize.py tests/test_gpu_determinism.py -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
timeout 300 python tools/step_launches.py 3 > /dev/null 2>&1 && \
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/step_launches.py 3 > /dev/null 2>&1; echo warm rc=$?
