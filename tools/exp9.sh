for mc in 1 2 3 4; do
TP_GEMM_KERNEL=2 TP_GEMM_MC=$mc python tools/gemm_bench.py --shapes 8192x8192x8192,512x4096x4096 --ops NN,TN --no-cublas --hot-graph | cut -c1-200 | sed "s/^/hot mc$mc /"
TP_GEMM_KERNEL=2 TP_GEMM_MC=$mc python tools/gemm_trace.py 8192x8192x8192 NN --hot | sed "s/^/trace mc$mc /"
done
TP_GEMM_KERNEL=2 TP_GEMM_MC=4 TP_GEMM_BN=128 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --no-cublas --hot-graph | cut -c1-200 | sed "s/^/hot mc4-128 /"
TP_GEMM_KERNEL=2 TP_GEMM_MC=4 python tools/gemm_trace.py 512x4096x4096 NN --hot | sed "s/^/trace mc4 512 /"
python tools/gemm_bench.py --shapes 8192x8192x8192 --ops NN --hot-graph | cut -c1-250 | sed "s/^/cublas /"
