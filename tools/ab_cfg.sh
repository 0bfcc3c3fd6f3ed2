# A/B of single-frame configs 3 and 2 (bench step time + per-kernel profile): tools/ab_cfg.sh V0 E1 ...
L=paper_2301_05262_b200/libnsm.so
cp $L /tmp/libnsm.keep
for X in "$@"; do
  cp tools/ab/$X.so $L
  for c in 3 2; do
  echo -n "$X cfg$c: "; timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-variants --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k: round(v*1000,1) for k,v in d['kernel_profile_ms_per_step'].items()})"
  done
done
cp /tmp/libnsm.keep $L
