# epilogue's tfull poll: nanosleep 200 vs 32 between try_waits (pair kernel)
for ns in 200 32; do
  sed -i "s/mbar_wait_sleep(&tfull\[acc\], acc_phase, [0-9]*)/mbar_wait_sleep(\&tfull[acc], acc_phase, $ns)/" paper_2110_14883_b200/csrc/gemm_sm100_2cta.cu
  python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
  echo "== sleep $ns"
  python tools/gemm_bench.py --shapes 16384x16384x64,4096x4096x512 --ops TN --iters 10 --no-cublas | cut -c1-110
  TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 8192x8192x8192 --ops NN --hot-graph --no-cublas | cut -c1-110
  for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'])"; done
done
