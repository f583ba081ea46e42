TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NT --hot | cut -c1-330 | sed "s/^/hot 4k NT /"
TP_GEMM_KERNEL=2 python tools/gemm_bench.py --shapes 8192x8192x8192,4096x4096x4096,512x4096x4096 --ops NN --hot-graph | cut -c1-250 | sed "s/^/hot /"
