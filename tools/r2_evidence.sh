# ncu evidence for profiles/ (run under gpurun): launch lists + --set full
# captures of the default (4-plane config 4) and the blocker (config 3) paths,
# traffic.json rows, then bench lines.  usage: bash tools/r2_evidence.sh TAG
set -x
T=${1:-r2x}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-soak --no-variants"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_cfg3.csv $B --config 3 > gpurun_out/ncu_l3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"enc0|level_kernel|dec0|recon" -c 10 -o gpurun_out/full -f $B --steps 1 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"feat5|enc0_s2d" -c 2 -o gpurun_out/full5 -f $B --steps 1 --features 5 > gpurun_out/ncu_full5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"feat5|enc0_s2d" -c 2 -o gpurun_out/full3 -f $B --steps 1 --config 3 > gpurun_out/ncu_full3.log 2>&1
ls -la gpurun_out
