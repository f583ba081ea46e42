timeout 900 python tools/trace_schedule.py --mode 3d --json gpurun_out/trace_3d.json > gpurun_out/trace_3d.txt 2>&1; tail -25 gpurun_out/trace_3d.txt
timeout 900 python tools/trace_schedule.py --mode 2d --json gpurun_out/trace_2d.json > gpurun_out/trace_2d.txt 2>&1; tail -25 gpurun_out/trace_2d.txt
timeout 1200 python -m pytest tests/test_gpu_c3head.py tests/test_gpu_tp.py tests/test_gpu_nccl.py -q -x > gpurun_out/r02_t19.log 2>&1; tail -3 gpurun_out/r02_t19.log
