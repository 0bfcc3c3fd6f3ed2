# quick: correctness subset + bench summary (args passed to bench.py)
timeout 300 python -m pytest tests/test_gpu_texels.py tests/test_gpu_f16.py -m gpu -q -x 2>&1 | tail -1
timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-variants "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac'], {k: round(v*1000,1) for k,v in d['kernel_profile_ms_per_step'].items()})"
