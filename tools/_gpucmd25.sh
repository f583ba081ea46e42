TP_GEMM_KERNEL=2 TP_GEMM_BN=128 TP_GEMM_MC=2 ncu --set full --clock-control none --import-source on -k regex:gemm -o gpurun_out/ncu_c2_mc2 python tools/ncu_shapes.py --only c2_fwd > /dev/null 2>&1; echo rc=$?
TP_GEMM_KERNEL=2 TP_GEMM_BN=128 TP_GEMM_MC=2 python tools/gemm_trace.py 512x4096x4096 NN --hot
TP_GEMM_KERNEL=2 TP_GEMM_BN=128 TP_GEMM_MC=2 python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --iters 50
python tools/gemm_bench.py --shapes 512x4096x4096 --ops NN --iters 50
