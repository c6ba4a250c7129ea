# A/B of environment switches on the config-3 bench (short runs, no CPU baseline)
cd $GRAFT_REPO_ROOT
for v in "" ${AB_VARIANTS}; do
  for rep in 1 2; do
    env $v timeout 300 python bench.py --steps 40 --no-cpu-baseline > gpurun_out/ab.json 2> gpurun_out/ab.err
    python -c "import json,sys;d=json.load(open('gpurun_out/ab.json'));k=d['roofline']['kernel_ms'];print(sys.argv[1] or 'base', d['value'], d['e2e']['value'], k['sb_blend_fwd'], k['sb_blend_bwd'])" "$v"
  done
done
