# where the 512-row pair GEMM spends its time (per-CTA trace), hot and cold
for bn in 128 256; do for h in "" "--hot"; do
 echo "BN=$bn $h: $(TP_GEMM_KERNEL=2 TP_GEMM_BN=$bn python tools/gemm_trace.py 512x4096x4096 NN $h 2>&1 | tail -1)"
done; done
echo "4096x4096x512: $(TP_GEMM_KERNEL=2 python tools/gemm_trace.py 4096x4096x512 NN --hot 2>&1 | tail -1)"
echo "8192^3: $(TP_GEMM_KERNEL=2 python tools/gemm_trace.py 8192x8192x8192 NN --hot 2>&1 | tail -1)"
