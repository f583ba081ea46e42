for d in 1 3 5 7; do
TP_GEMM_DBG=$d TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NN --hot | cut -c1-330 | sed "s/^/dbg$d hot 4k NN /"
TP_GEMM_DBG=$d TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NT --hot | cut -c1-330 | sed "s/^/dbg$d hot 4k NT /"
done
