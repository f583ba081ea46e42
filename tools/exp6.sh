for k in 1 2; do
TP_GEMM_KERNEL=$k python tools/gemm_bench.py --shapes 512x4096x4096,4096x4096x512,512x4096x16384 --ops NN --no-cublas --hot-graph | cut -c1-140 | sed "s/^/hot k$k /"
TP_GEMM_KERNEL=$k python tools/gemm_bench.py --shapes 512x4096x16384 --ops NN --no-cublas | cut -c1-140 | sed "s/^/cold k$k /"
done
python tools/gemm_bench.py --shapes 512x4096x4096,512x4096x16384 --ops NN --hot-graph | cut -c1-240 | sed "s/^/hot cublas-cmp /"
