# per-change gate: GPU tests (-x), warm-cache launch list, one short bench line
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
grep -E "passed|failed|error" gpurun_out/pytest_gpu.log | tail -3
timeout 300 python tools/step_launches.py 3 > /dev/null 2>&1 && \
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/step_launches.py 3 > /dev/null 2>&1; echo warm rc=$?
timeout 900 python bench.py --steps 30 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "full", d["full_lists"]["value"], "atomic", d["atomic_backward"]["value"], "fps", d["render_fps"], "noskip", d.get("no_touched_skip", {}).get("value"))
print("batched", d.get("batched", {}).get("value"), d.get("batched", {}).get("e2e", {}).get("value"))
print(d["roofline"]["kernel_ms"])
PY
