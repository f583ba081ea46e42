# default dispatch vs every GEMM on the pair kernel, C2
for k in 0 2; do for r in 1 2; do TP_GEMM_KERNEL=$k python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('kernel=$k c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done; done
