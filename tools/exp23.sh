TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 8192x8192x8192,4096x4096x4096,512x4096x4096,4096x4096x512 --ops NN,NT,TN --hot-graph 2>&1 | cut -c1-250
python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512 --ops NN,NT,TN 2>&1 | cut -c1-250 | sed "s/^/auto cold /"
