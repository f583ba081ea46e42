timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
for mc in 1 2; do for bn in 128 256; do
TP_GEMM_MC=$mc TP_GEMM_BN=$bn python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN,TN --no-cublas | cut -c1-150 | sed "s/^/mc$mc bn$bn /"
done; done
for mc in 1 2; do
TP_GEMM_MC=$mc python tools/gemm_bench.py --shapes 4096x4096x512,8192x8192x8192 --ops NN,NT,TN --no-cublas | cut -c1-150 | sed "s/^/mc$mc auto /"
done
