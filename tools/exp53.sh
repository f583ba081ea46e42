# 1-CTA GEMM: TMA-store epilogue (smem staging) vs direct row stores
timeout 1500 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x 2>&1 | tail -1
for t in 1 0; do
  echo "== TMA store $t"
  TP_GEMM_V1_TMA_STORE=$t TP_GEMM_KERNEL=1 python tools/gemm_bench.py --shapes 512x4096x4096,64x16384x16384 --ops NN --hot-graph --no-cublas | cut -c1-120
  for r in 1 2; do TP_GEMM_V1_TMA_STORE=$t python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
  TP_GEMM_V1_TMA_STORE=$t python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['roofline']['frac'])"
done
