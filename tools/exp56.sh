# split-K of two as a reduce-scatter between the two co-resident splits
timeout 1500 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -1
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT --hot-graph --no-cublas | cut -c1-110
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --no-cublas | cut -c1-110
echo "trace: $(TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_trace.py 512x4096x4096 NN --hot 2>&1 | tail -1 | cut -c1-330)"
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
for r in 1 2; do TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 pair256', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
