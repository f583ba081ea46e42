# explicit st.shared for the GEMM epilogue staging and the flash P tile / max exchange
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py tests/test_gpu_fused.py -m gpu -q -x 2>&1 | tail -1
python tools/gemm_bench.py --shapes 16384x16384x64,4096x4096x512 --ops TN --iters 10 --no-cublas | cut -c1-130
TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 4096x4096x512,512x4096x4096,8192x8192x8192 --ops NN --hot-graph --no-cublas | cut -c1-130
for r in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['ms_per_step'], d['roofline']['achieved'])"; done
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['roofline']['frac'])"
for cfg in "8192 128 16" "16384 128 8" "8192 64 16"; do echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1 | cut -c1-130)"; done
