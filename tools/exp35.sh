# flash softmax: unpredicated full tiles, ex2.approx, 8-way max / sum chains; all heads per ring launch
timeout 900 python -m pytest tests/test_gpu_rsa.py tests/test_gpu_flash.py tests/test_gpu_attention.py tests/test_gpu_block.py -m gpu -q 2>&1 | tail -3
for cfg in "8192 64 16" "8192 128 16" "16384 128 8" "2048 64 64"; do
  echo "$cfg: $(python tools/rsa_bench.py $cfg 2>&1 | tail -1)"
done
ncu --set full --import-source on --clock-control none -k regex:flash_fwd -c 1 -o gpurun_out/flash_full2 python tools/rsa_bench.py 8192 64 16 > /dev/null 2>&1
