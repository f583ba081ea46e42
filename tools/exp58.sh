# flash d = 64: K / V ring of 3 stages vs 2
for kv in 3 2; do
  sed -i "s/^#define TP_FLASH_KV64 [0-9]/#define TP_FLASH_KV64 $kv/" paper_2110_14883_b200/csrc/flash.cu
  python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
  echo "== KV64=$kv"
  for cfg in "8192 64 16" "16384 64 8" "2048 64 64"; do echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1 | cut -c1-130)"; done
done
sed -i "s/^#define TP_FLASH_KV64 [0-9]/#define TP_FLASH_KV64 3/" paper_2110_14883_b200/csrc/flash.cu
python -c "from paper_2110_14883_b200 import build as b; b.build()" 2>&1 | grep -i error
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py tests/test_gpu_block.py -m gpu -q 2>&1 | tail -1
