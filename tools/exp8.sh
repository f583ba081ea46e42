S=512x4096x4096
for bn in 256 128; do for sp in 0 1; do
TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn TP_GEMM_SPLITK=$sp python tools/gemm_trace.py $S NN | sed "s/^/cold pair-$bn-split$sp /"
TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn TP_GEMM_SPLITK=$sp python tools/gemm_trace.py $S NN --hot | sed "s/^/hot pair-$bn-split$sp /"
done; done
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 8192x8192x8192 NN --hot | sed "s/^/hot pair-8k /"
