# split-K owner pipeline (per-warp 64-column flags) on the 512-row GEMMs
timeout 1200 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -2
for bn in 256 128; do echo "BN=$bn: $(TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn python tools/gemm_trace.py 512x4096x4096 NN --hot 2>&1 | tail -1 | cut -c1-420)"; done
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT,TN --hot-graph | cut -c1-200
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --no-cublas | cut -c1-200
python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --no-cublas | cut -c1-200
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
