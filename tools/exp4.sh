timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
TP_GEMM_MC=3 timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -k "gemm" 2>&1 | tail -2
for mc in 1 3; do for bn in 128 256; do
TP_GEMM_MC=$mc TP_GEMM_BN=$bn python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,NT,TN --no-cublas | cut -c1-130 | sed "s/^/mc$mc bn$bn /"
done; done
TP_GEMM_MC=3 TP_GEMM_BN=128 python tools/gemm_trace.py 512x4096x4096 NN
