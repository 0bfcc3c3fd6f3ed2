mkdir -p gpurun_out
[ -n "$SKIPT" ] || timeout 400 python -m pytest tests/test_gpu_blocker5.py -m gpu -q -rf -x > gpurun_out/pytest_c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_c.log
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-variants "$@" > gpurun_out/bench_c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c.log
tail -4 gpurun_out/pytest_c.log
python - <<PY
import json
for l in open('gpurun_out/bench_c.log'):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], {k: round(v*1000,1) for k,v in d['kernel_profile_ms_per_step'].items()})
PY
tail -2 gpurun_out/bench_c.log | cut -c1-300
