# round-end evidence: GPU suite, smoke, the default bench line and its
# reference arm, configs 4 and 5, warm and cold launch lists, one full
# capture of the step's kernels (each ncu pass only after its program ran
# clean without ncu), the config-5 batch launch list
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench rc=$?
timeout 1200 python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo ref rc=$?
timeout 900 python tools/stream_bench.py > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; echo c4 rc=$?
timeout 900 python bench.py --batched --config 5 --steps 10 --warmup 3 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err; echo c5 rc=$?
timeout 300 python tools/step_launches.py 3 > /dev/null 2>&1 && \
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_warm.csv python tools/step_launches.py 3 > /dev/null 2>&1; echo warm rc=$?
bash tools/gpu_r2_evidence.sh
timeout 300 python tools/batch_launches.py > /dev/null 2>&1 && \
timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_c5_launches.csv python tools/batch_launches.py 1 > /dev/null 2>&1; echo c5 launches rc=$?
SB_PROFILE_TAIL=1 timeout 900 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_c4_launches.csv python tools/stream_bench.py > /dev/null 2>&1; echo c4 launches rc=$?
