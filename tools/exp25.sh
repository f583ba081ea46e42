TP_GEMM_KERNEL=2 python tools/gemm_trace.py 512x4096x4096 NN --hot | cut -c1-600
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 512x4096x4096 NN | cut -c1-600
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_trace.py 512x4096x4096 NN --hot | cut -c1-600
