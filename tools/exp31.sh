# SIMT-coalesced epilogue (TP_GEMM_EPI=1) vs TMA-store epilogue (0) on the CTA-pair GEMM
TP_GEMM_EPI=1 timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_fused.py -m gpu -q -x 2>&1 | tail -2
for e in 0 1; do
  echo "== EPI=$e pair default"
  TP_GEMM_EPI=$e TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,512x4096x4096,8192x8192x8192 --ops NN,TN --hot-graph --no-cublas | cut -c1-110
  echo "== EPI=$e pair BN=256 (split-K on 512 rows)"
  TP_GEMM_EPI=$e TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT --hot-graph --no-cublas | cut -c1-110
  TP_GEMM_EPI=$e python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"
done
