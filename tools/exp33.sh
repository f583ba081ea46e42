# online-softmax RSA ring: parity, then fused vs two-pass timing; bench e2e
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py -m gpu -q 2>&1 | tail -4
for f in 1 0; do
  for cfg in "8192 64 16" "8192 128 16" "16384 128 8" "2048 64 64"; do
    echo "TP_RSA_FUSED=$f $cfg: $(TP_RSA_FUSED=$f python tools/rsa_bench.py $cfg 2>&1 | tail -1)"
  done
done
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; cat gpurun_out/bench_e2e.json
