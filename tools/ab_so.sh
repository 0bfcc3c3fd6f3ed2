# A/B of prebuilt library variants on one box: tools/ab/lib<X>.so swapped in
# as libnsm.so, interleaved, each a short bench (value, ms/step, enc0 us)
for r in 1 2; do
for v in "$@"; do
cp tools/ab/lib$v.so paper_2301_05262_b200/libnsm.so
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-soak 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_profile_ms_per_step']
print('$v', d['value'], d['ms_per_step'], ' '.join(f'{n}={x*1000:.1f}' for n,x in k.items()))"
done
done
