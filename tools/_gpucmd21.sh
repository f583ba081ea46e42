timeout 900 python -m pytest tests/test_gpu_attention.py tests/test_gpu_block.py tests/test_gpu_block_widths.py tests/test_gpu_rsa.py tests/test_gpu_flash.py -q -x > gpurun_out/r02_t21.log 2>&1; tail -4 gpurun_out/r02_t21.log
timeout 300 python tools/attn_bench.py --seq 2048 --batch 8 --heads 64 --dh 128
timeout 300 python tools/attn_bench.py --seq 8192 --batch 1 --heads 16 --dh 128
timeout 300 python tools/attn_bench.py --seq 197 --batch 512 --heads 6 --dh 64
timeout 300 python tools/attn_bench.py --seq 8192 --batch 1 --heads 16 --dh 64
timeout 300 python tools/transformer_bench.py --workload c5
