for v in 1 0 1 0; do
NSM_DEC0_RING=$v python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ring=$v', d['value'], d['ms_per_step'])"
done
