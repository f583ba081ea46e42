# fraction of the softmax exponentials computed by a polynomial on the FMA pipe
for n in 4 2 8 0; do
  sed -i "s/^#define TP_FLASH_POLY_EVERY [0-9]*/#define TP_FLASH_POLY_EVERY $n/" paper_2110_14883_b200/csrc/flash.cu
  python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
  echo "== every $n"
  for cfg in "8192 64 16" "8192 128 16"; do echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1 | cut -c1-160)"; done
done
sed -i "s/^#define TP_FLASH_POLY_EVERY [0-9]*/#define TP_FLASH_POLY_EVERY 4/" paper_2110_14883_b200/csrc/flash.cu
python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py -m gpu -q 2>&1 | tail -1
