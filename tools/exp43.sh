# flash d=64 with 8 softmax warps (two per TMEM lane quadrant, 64 keys each)
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py tests/test_gpu_block.py -m gpu -q 2>&1 | tail -3
for cfg in "8192 64 16" "8192 128 16" "2048 64 64" "16384 64 8"; do
  echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1)"
done
