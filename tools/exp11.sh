TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NN --hot | sed "s/^/hot 4k NN /"
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 8192x8192x8192 NN --hot | sed "s/^/hot 8k NN /"
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 512x4096x4096 NN --hot | sed "s/^/hot 512 NN /"
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_trace.py 512x4096x4096 NN --hot | sed "s/^/hot 512 NN bn256 /"
