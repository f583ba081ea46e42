TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NN --hot | cut -c1-400 | sed "s/^/hot 4k NN /"
TP_GEMM_DBG=7 TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NT --hot | cut -c1-400 | sed "s/^/dbg7 hot 4k NT /"
