python -m pytest tests/test_gpu_f16.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for pdl in 1 0 1; do
NSM_PDL=$pdl python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$pdl', d['value'], d['ms_per_step'], d['clocks'])"
done
