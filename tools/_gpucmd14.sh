timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "wide_pair" > gpurun_out/r02_t14a.log 2>&1; tail -3 gpurun_out/r02_t14a.log
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x -k "variants_forced and WIDE" > gpurun_out/r02_t14b.log 2>&1; tail -3 gpurun_out/r02_t14b.log
for w in 0 1; do echo "wide $w"; TP_GEMM_WIDE=$w timeout 300 python tools/gemm_bench.py --shapes 16384x16384x16384,8192x8192x8192 --ops NN,NT,TN --iters 40 2>&1 | tail -6; done
timeout 900 python -m pytest tests/test_gpu_c3head.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r02_t14c.log 2>&1; tail -3 gpurun_out/r02_t14c.log
for w in 1 0; do TP_GEMM_WIDE=$w python bench.py --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_wide$w.json 2>&1; python -c "import json;d=json.load(open('gpurun_out/r02_bench_wide$w.json'));print('bench wide $w', d['value'], d['ms_per_step'], d['clocks'])"; done
