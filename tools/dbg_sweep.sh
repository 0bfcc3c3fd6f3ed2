# Bottleneck attribution: per-kernel times with parts of each kernel skipped
# (experiment switches NSM_*_DBG; results are wrong by construction).
for v in "" "NSM_ENC0_DBG=1" "NSM_ENC0_DBG=2" "NSM_ENC0_DBG=3" "NSM_LEVEL_DBG=1" "NSM_LEVEL_DBG=2" "NSM_LEVEL_DBG=4" "NSM_LEVEL_DBG=6"; do
  env $v python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-soak 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); k=d['kernel_profile_ms_per_step']
print('$v'.ljust(18), ' '.join(f'{n}={v*1000:.0f}' for n,v in k.items()))"
done
