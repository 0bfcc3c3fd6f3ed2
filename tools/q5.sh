# quick 5-plane check: blocker tests + bench config 4 (5 planes) and config 3
timeout 400 python -m pytest tests/test_gpu_blocker5.py -m gpu -q -x 2>&1 | tail -1
for a in "--features 5" "--config 3"; do
timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-variants $a 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$a', d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], {k: round(v*1000,1) for k,v in list(d['kernel_profile_ms_per_step'].items())[:3]})"
done
