for d in 0 1; do
TP_GEMM_DBG=$d TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NN --hot | sed "s/^/dbg$d hot 4k NN /"
TP_GEMM_DBG=$d TP_GEMM_KERNEL=2 TP_GEMM_BN=256 TP_GEMM_SPLITK=0 python tools/gemm_trace.py 512x4096x4096 NN --hot | sed "s/^/dbg$d hot 512 NN bn256 /"
done
