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
