# quick GPU check: GPU tests + a short bench line summary (test result last)
T=$(python -m pytest tests -m gpu -x -q 2>&1 | tail -1)
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'], {k: round(v*1000,1) for k,v in d['kernel_profile_ms_per_step'].items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])"
echo "TESTS: $T"
