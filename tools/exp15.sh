for d in 1 9; do
TP_GEMM_DBG=$d TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NT --hot | cut -c1-300 | sed "s/^/dbg$d hot 4k NT /"
TP_GEMM_DBG=$d TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x8192 NT --hot | cut -c1-300 | sed "s/^/dbg$d hot 4kx8k NT /"
done
