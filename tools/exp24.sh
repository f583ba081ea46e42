for k in 1 2; do
TP_GEMM_KERNEL=$k python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512,1024x4096x4096,8192x8192x8192 --ops NN,NT,TN --no-cublas 2>&1 | cut -c1-160 | sed "s/^/cold k$k /"
TP_GEMM_KERNEL=$k python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512 --ops NN --no-cublas --hot-graph 2>&1 | cut -c1-160 | sed "s/^/hot k$k /"
done
TP_GEMM_KERNEL=1 TP_GEMM_V1_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512 --ops NN --no-cublas 2>&1 | cut -c1-160 | sed "s/^/cold k1-256 /"
TP_GEMM_KERNEL=2 TP_GEMM_BN=128 python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512 --ops NN --no-cublas 2>&1 | cut -c1-160 | sed "s/^/cold k2-128 /"
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512 --ops NN --no-cublas 2>&1 | cut -c1-160 | sed "s/^/cold k2-256 /"
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 TP_GEMM_SPLITK=0 python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512 --ops NN --no-cublas 2>&1 | cut -c1-160 | sed "s/^/cold k2-256-nosplit /"
