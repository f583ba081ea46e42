# epilogue warps 4 vs 8 (two per TMEM lane quadrant) after the tempty fence fix
run() {
  python tools/gemm_bench.py --shapes 16384x16384x64 --ops TN --iters 10 --no-cublas | cut -c1-130
  TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,512x4096x4096,8192x8192x8192 --ops NN --hot-graph --no-cublas | cut -c1-130
  for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
  python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['roofline']['frac'])"
  python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', d['value'], d['roofline']['frac'])"
}
echo "== 4 epilogue warps"; run
sed -i 's/^#define TP_EPI_WARPS 4$/#define TP_EPI_WARPS 8/' paper_2110_14883_b200/csrc/gemm_sm100_2cta.cu
python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
echo "== 8 epilogue warps"; run
timeout 900 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "not forced" 2>&1 | tail -1
