for pdl in 1 0; do
TP_PDL=$pdl TP_GEMM_KERNEL=2 TP_GEMM_BN=256 TP_GEMM_SPLITK=0 python tools/gemm_trace.py 512x4096x4096 NT --hot | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pdl$pdl 512 NT', {k:d[k] for k in ['steady_cyc_per_kb','cta_us','sm_mhz']})"
done
