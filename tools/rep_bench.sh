# repeated short bench lines (value, ms/step) for A/B decisions
for i in 1 2 3; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-soak "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])"
done
