# Epilogue variants of the CTA-pair GEMM (TP_GEMM_EPI 0/1/2): correctness + timing
set -x
for e in 1 2; do TP_GEMM_EPI=$e timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py -m gpu -q -x 2>&1 | tail -3; done
for e in 0 1 2; do
  echo "== EPI=$e"
  TP_GEMM_EPI=$e TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,512x4096x4096,8192x8192x8192 --ops NN,TN --hot-graph --no-cublas | cut -c1-300
  TP_GEMM_EPI=$e python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
done
