# d = 128 with eight softmax warps and a single P buffer (TP_FLASH_W128=1) vs four warps, two P buffers
for w in 1 0; do
  sed -i "s/^#define TP_FLASH_W128 [0-9]/#define TP_FLASH_W128 $w/" paper_2110_14883_b200/csrc/flash.cu
  python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
  echo "== W128=$w"
  for cfg in "8192 128 16" "16384 128 8" "2048 128 64" "8192 64 16"; do echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1 | cut -c1-160)"; done
  timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py tests/test_gpu_block.py -m gpu -q 2>&1 | tail -1
done
