for bn in 128 256; do
TP_GEMM_KERNEL=1 TP_GEMM_V1_BN=$bn python tools/gemm_bench.py --shapes 512x4096x4096,1024x4096x4096,4096x4096x512 --ops NN,NT,TN --no-cublas | cut -c1-130 | sed "s/^/v1 bn$bn /"
done
python tools/gemm_bench.py --shapes 1024x4096x4096,2048x4096x4096 --ops NN --no-cublas | cut -c1-130 | sed "s/^/pair /"
