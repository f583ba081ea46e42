TP_GEMM_KERNEL=2 TP_GEMM_MC=5 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096,1024x4096x4096 --ops NN,NT,TN --no-cublas --hot-graph | cut -c1-130 | sed "s/^/hot mc5 /"
TP_GEMM_KERNEL=2 TP_GEMM_MC=5 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT,TN --no-cublas | cut -c1-130 | sed "s/^/cold mc5 /"
TP_GEMM_KERNEL=2 TP_GEMM_MC=5 python tools/gemm_trace.py 512x4096x4096 NN --hot | cut -c1-600
