TP_NVCC_FLAGS=-DTP_LOOP_CLOCKS=1 python -m paper_2110_14883_b200.build --force -j 16 > /dev/null 2>&1; echo build=$?
for mc in 1 2; do TP_GEMM_KERNEL=2 TP_GEMM_BN=128 TP_GEMM_MC=$mc python tools/gemm_trace.py 512x4096x4096 NN --hot; done
TP_GEMM_KERNEL=2 TP_GEMM_BN=256 python tools/gemm_trace.py 8192x8192x8192 NN --hot
