# flash d = 64 as two CTAs per SM (4 softmax warps, single S / P / K-V buffers) vs one CTA with 8 warps
for t in 1 0; do
  sed -i "s/^#define TP_FLASH_2CTA64 [0-9]/#define TP_FLASH_2CTA64 $t/" paper_2110_14883_b200/csrc/flash.cu
  python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
  echo "== 2CTA64=$t"
  for cfg in "8192 64 16" "16384 64 8" "2048 64 64"; do echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1 | cut -c1-130)"; done
  timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py -m gpu -q 2>&1 | tail -1
done
