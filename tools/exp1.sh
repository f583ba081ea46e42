S=512x4096x4096
for pf in 0 4 8 16; do
  TP_GEMM_PREFETCH=$pf python tools/gemm_bench.py --shapes $S --ops NN --no-cublas
  TP_GEMM_PREFETCH=$pf python tools/gemm_bench.py --shapes $S --ops NN --no-cublas --no-split
done
python tools/gemm_bench.py --shapes $S --ops NN --no-flush
python tools/gemm_bench.py --shapes $S --ops NN --no-flush --no-split
TP_GEMM_KERNEL=1 python tools/gemm_bench.py --shapes $S --ops NN --no-flush
TP_GEMM_PREFETCH=8 python tools/gemm_bench.py --shapes 4096x4096x512,8192x8192x8192 --ops NN,TN --no-cublas
