for d in randn zeros ones uniform ternary; do
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 TP_GEMM_SPLITK=0 python tools/gemm_trace.py 512x4096x4096 NT --hot --data=$d | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d 512 NT', {k:d[k] for k in ['steady_cyc_per_kb','cta_us','sm_mhz']})"
TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x4096 NT --hot --data=$d | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$d 4k NT', {k:d[k] for k in ['steady_cyc_per_kb','cta_us','sm_mhz']})"
done
