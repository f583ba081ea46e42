# TMEM hand-back (tempty) arrive / wait at CTA-scope semantics instead of .release/.acquire.cluster
timeout 1200 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -2
python tools/gemm_bench.py --shapes 16384x16384x64 --ops TN --iters 10 | cut -c1-250
TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,512x4096x4096,8192x8192x8192 --ops NN,TN --hot-graph --no-cublas | cut -c1-120
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'])"
