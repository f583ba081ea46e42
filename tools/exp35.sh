# flash: double-buffered P + lazy rescale (softmax a tile ahead of the PV MMA)
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py tests/test_gpu_block.py -m gpu -q 2>&1 | tail -3
for cfg in "8192 64 16" "8192 128 16" "16384 128 8" "2048 64 64"; do
  echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1)"
done
ncu --set full --import-source on --clock-control none -k regex:flash_fwd -c 1 -o gpurun_out/flash_full3 python tools/rsa_bench.py 8192 64 16 > /dev/null 2>&1
