# pair GEMM epilogue tail: wait_group.read instead of full completion
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py tests/test_gpu_tp.py -m gpu -q -x 2>&1 | tail -2
for bn in 128 256; do echo "BN=$bn: $(TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn python tools/gemm_trace.py 512x4096x4096 NN --hot 2>&1 | tail -1 | cut -c1-400)"; done
TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,512x4096x4096 --ops NN,TN --hot-graph --no-cublas | cut -c1-120
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
