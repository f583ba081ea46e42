# split-K partial hand-off: fence.acq_rel.gpu instead of __threadfence (fence.sc.gpu)
timeout 1500 python -m pytest tests/test_gpu_kernels.py -m gpu -q -x -k "split or pair or deterministic or forced" 2>&1 | tail -1
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --hot-graph --no-cublas | cut -c1-110
for r in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
