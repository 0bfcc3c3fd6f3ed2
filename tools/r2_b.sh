mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_blocker5.py tests/test_gpu_texels.py tests/test_gpu_f16.py tests/test_gpu_parity.py -m gpu -q -rf -x > gpurun_out/pytest_b.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_b.log
timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench5.log 2>&1; echo "rc=$?" >> gpurun_out/bench5.log
timeout 120 python bench.py --features 4 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
tail -15 gpurun_out/pytest_b.log
for f in bench5 bench4; do python - <<PY
import json
for l in open('gpurun_out/$f.log'):
    if l.startswith('{'):
        d=json.loads(l); print('$f', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], {k: round(v*1000,1) for k,v in d['kernel_profile_ms_per_step'].items()}, d['variants'])
PY
tail -3 gpurun_out/$f.log | cut -c1-300; done
