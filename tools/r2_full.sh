# Full GPU pass: all GPU tests, smoke, bench configs 4 (default), 3, 5.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py > gpurun_out/bench.log 2>&1; echo "rc=$?" >> gpurun_out/bench.log
timeout 300 python bench.py --config 3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg3.log
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1; echo "rc=$?" >> gpurun_out/bench_cfg5.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref.log
tail -8 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log
for f in bench bench_cfg3 bench_cfg5 bench_ref; do echo "== $f"; tail -2 gpurun_out/$f.log | cut -c1-600; done
