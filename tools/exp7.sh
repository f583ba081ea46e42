# small-M GEMM variant sweep (512x4096x4096 NN and NT, 4096x4096x512 TN), cold (L2 flushed) and hot
S=512x4096x4096
for hot in "" "--hot-graph"; do
python tools/gemm_bench.py --shapes $S,4096x4096x512 --ops NN,NT,TN $hot | cut -c1-260 | sed "s/^/auto $hot /"
TP_GEMM_KERNEL=1 TP_GEMM_V1_BN=128 python tools/gemm_bench.py --shapes $S --ops NN --no-cublas $hot | cut -c1-160 | sed "s/^/v1-128 $hot /"
TP_GEMM_KERNEL=1 TP_GEMM_V1_BN=256 python tools/gemm_bench.py --shapes $S --ops NN --no-cublas $hot | cut -c1-160 | sed "s/^/v1-256 $hot /"
for bn in 256 128; do for sp in 0 1; do
TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn TP_GEMM_SPLITK=$sp python tools/gemm_bench.py --shapes $S --ops NN --no-cublas $hot | cut -c1-160 | sed "s/^/pair-$bn-split$sp $hot /"
done; done
done
for bn in 256 128; do for sp in 0 1; do
TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn TP_GEMM_SPLITK=$sp python tools/gemm_trace.py $S NN | sed "s/^/trace pair-$bn-split$sp /"
done; done
