# quick GPU check: fp16 parity tests + a short bench line summary
python -m pytest tests/test_gpu_f16.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['kernel_profile_ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
