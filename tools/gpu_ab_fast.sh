cd $GRAFT_REPO_ROOT
for t in . _ab/fast; do
  name=$(echo $t | tr '/.' '__')
  (cd $t && timeout 300 python tools/step_launches.py 3 > /dev/null 2>&1 && \
   timeout 600 ncu --profile-from-start off --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file $GRAFT_REPO_ROOT/gpurun_out/warm_$name.csv python tools/step_launches.py 3 > /dev/null 2>&1; echo $t rc=$?)
  (cd $t && timeout 600 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-batched > $GRAFT_REPO_ROOT/gpurun_out/bench_$name.json 2>/dev/null; echo bench rc=$?)
done
