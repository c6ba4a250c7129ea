# after tools/gpu_final.sh: summarise its outputs into profiles/ (round 2)
set -e
cd "$(dirname "$0")/.."
python tools/ncu_json.py gpurun_out/r2_full.ncu-rep 3 r2 > /dev/null
python tools/ncu_summary.py full gpurun_out/r2_full.ncu-rep > profiles/r2_kernels.md
python tools/ncu_summary.py launches gpurun_out/r2_launches.csv 3 > profiles/r2_launches.md
python tools/ncu_summary.py launches gpurun_out/final_launches_warm.csv 3 > profiles/r2_launches_warm.md
sed -i 's/^Cold-cache, serialised per-launch times (`--clock-control none`): compare SHARES./Warm-cache (`--cache-control none --clock-control none`), serialised per-launch times of tools\/step_launches.py (DRAM columns not collected in this pass): compare SHARES./' profiles/r2_launches_warm.md
python tools/ncu_summary.py launches gpurun_out/final_c5_launches.csv 1 > profiles/r2_config5_launches.md
sed -i 's/^# ncu launch list (\([0-9]*\) launches; 1 steps incl. warm-up\/e2e\/timing passes)/# ncu launch list of one config-5 batch (\1 launches: 8 views + exchange + Adam, tools\/batch_launches.py, eager)/; s/^Cold-cache, serialised per-launch times (`--clock-control none`): compare SHARES./Warm-cache (`--cache-control none --clock-control none`), serialised per-launch times (DRAM columns not collected): compare SHARES./' profiles/r2_config5_launches.md
tail -n1 gpurun_out/final_c4.json > profiles/r2_config4_stream.json
tail -n1 gpurun_out/final_c5.json > profiles/r2_config5_batched.json
tail -n1 gpurun_out/final_bench.json > profiles/r2_bench.json
tail -n1 gpurun_out/final_bench_ref.json > profiles/r2_bench_reference.json
{ echo "# config-4 full-size map (4.04M rows, after the 1000-frame stream): 3 eager steps of the last keyframe (tools/stream_bench.py, SB_PROFILE_TAIL=1)"; echo
  python tools/ncu_summary.py launches gpurun_out/final_c4_launches.csv 3 | tail -n +2 | sed 's/^Cold-cache, serialised per-launch times (`--clock-control none`): compare SHARES./Warm-cache (`--cache-control none --clock-control none`), serialised per-launch times (DRAM columns not collected): compare SHARES./'
  echo; echo "Before the warp-cooperative big-row count and the warp-per-rank long gather (round 2, late): \`count_hist_kernel\` 983.2 us and \`gather_long_kernel\` 238.6 us per launch (26.4 % and 6.4 % of the step)."; } > profiles/r2_config4_launches.md
