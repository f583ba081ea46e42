# dispatch: pair 256x128 tiles for the 512-row products
for r in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
for w in c4 c3; do python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
