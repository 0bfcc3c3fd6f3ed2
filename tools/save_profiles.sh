# Copy a tools/gpu_round.sh result from gpurun_out/ into profiles/ under a tag.
# usage: bash tools/save_profiles.sh r1c
set -e
t=$1
cp gpurun_out/launches.csv profiles/${t}_launches.csv
python tools/ncu_summary.py full gpurun_out/full.ncu-rep profiles/${t}_full.json > profiles/${t}_full.md
python tools/ncu_summary.py launches gpurun_out/launches.csv > profiles/${t}_launches.md
python tools/ncu_stalls.py gpurun_out/full.ncu-rep 25 enc0 > profiles/${t}_enc0_stalls.txt || true
grep '^{' gpurun_out/bench.log | tail -1 > profiles/${t}_bench.json
grep '^{' gpurun_out/bench_ref.log | tail -1 > profiles/${t}_bench_ref.json
tail -3 gpurun_out/pytest_gpu.log > profiles/${t}_pytest_gpu.txt
cp gpurun_out/smoke.log profiles/${t}_smoke.txt
cp gpurun_out/traffic.json profiles/traffic.json
