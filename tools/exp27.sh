for mc in 1 5; do
TP_GEMM_KERNEL=2 TP_GEMM_MC=$mc TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096,1024x4096x4096,4096x4096x512 --ops NN,NT,TN --no-cublas --hot-graph | cut -c1-130 | sed "s/^/hot mc$mc /"
TP_GEMM_KERNEL=2 TP_GEMM_MC=$mc TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT --no-cublas | cut -c1-130 | sed "s/^/cold mc$mc /"
done
TP_GEMM_KERNEL=1 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --no-cublas | cut -c1-130 | sed "s/^/cold v1 /"
TP_GEMM_KERNEL=2 TP_GEMM_MC=5 python tools/gemm_trace.py 512x4096x4096 NN --hot | cut -c1-600
