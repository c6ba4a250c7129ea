# the deterministic backward: GPU tests, launch lists (cold- and warm-cache), bench
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
timeout 300 python tools/step_launches.py 3 > gpurun_out/sl_plain_0.log 2>&1 && \
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_atomic0.csv python tools/step_launches.py 3 > gpurun_out/sl_ncu_0.log 2>&1; echo cold rc=$?
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/step_launches.py 3 > gpurun_out/sl_ncu_w.log 2>&1; echo warm rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print('value', d['value'], 'e2e', d['e2e']['value'], 'fps', d['render_fps']); print(d['roofline']['kernel_ms'])"
