# A/B with the per-kernel profile: tools/ab/<X>.so swapped in, bench.py's kernel_profile_ms_per_step (config 4)
L=paper_2301_05262_b200/libnsm.so
cp $L /tmp/libnsm.keep
for X in "$@"; do
  cp tools/ab/$X.so $L
  echo -n "$X: "; timeout 300 python bench.py --steps 10 --warmup 3 --no-variants --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k: round(v*1000,1) for k,v in d['kernel_profile_ms_per_step'].items()})"
done
cp /tmp/libnsm.keep $L
