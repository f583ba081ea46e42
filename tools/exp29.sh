TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,4096x4096x1024,8192x8192x8192,512x4096x4096 --ops NN,TN --hot-graph | cut -c1-250
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['ms_per_step'])"
