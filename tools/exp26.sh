for own in 1 0; do
TP_GEMM_SPLIT_OWNER=$own TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_trace.py 512x4096x4096 NN --hot | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print('own$own', {k:d[k] for k in ['ctas','event_us','span_us','cta_us','exit_spread_us','sm_mhz','mma_total','epi_total']})"
TP_GEMM_SPLIT_OWNER=$own TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096,1024x4096x4096,512x8192x8192,256x4096x4096 --ops NN,NT,TN --no-cublas --hot-graph | cut -c1-150 | sed "s/^/hot own$own /"
TP_GEMM_SPLIT_OWNER=$own TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT,TN --no-cublas | cut -c1-150 | sed "s/^/cold own$own /"
done
