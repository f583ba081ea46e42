# per-problem epilogue warps (8 for <= 2 k-blocks per tile)
timeout 1500 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -1
python tools/gemm_bench.py --shapes 16384x16384x64,4096x4096x512 --ops TN --iters 10 --no-cublas | cut -c1-130
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['roofline']['frac'])"
python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['roofline']['frac'])"
