# Full GPU evidence pass (run under gpurun): tests, smoke, bench (both arms),
# ncu launch list + full capture of the fused-path kernels, traffic.json,
# then the final bench line with roofline.traffic filled from that capture.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pre.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-soak > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"enc0|level_kernel|dec0|recon" -c 10 -o gpurun_out/full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-soak > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py traffic gpurun_out/full.ncu-rep 8 profiles/traffic.json "ncu --set full, first launch (8 frames), $(date -u +%F)" > gpurun_out/traffic.log 2>&1 && cp profiles/traffic.json gpurun_out/traffic.json
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
ls -la gpurun_out
