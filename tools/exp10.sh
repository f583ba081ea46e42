for sp in 0 1; do
TP_GEMM_KERNEL=2 TP_GEMM_SPLITK=$sp python tools/gemm_trace.py 512x4096x4096 NN --hot | sed "s/^/hot 512 split$sp /"
TP_GEMM_KERNEL=2 TP_GEMM_SPLITK=$sp python tools/gemm_trace.py 512x4096x4096 NT --hot | sed "s/^/hot 512 NT split$sp /"
done
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 8192x8192x8192 NN --hot | sed "s/^/hot 8k NN /"
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 8192x8192x8192 NT --hot | sed "s/^/hot 8k NT /"
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NT --hot | sed "s/^/hot 4k NT /"
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NN --hot | sed "s/^/hot 4k NN /"
