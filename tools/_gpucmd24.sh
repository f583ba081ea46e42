for rep in 1 2; do for np in 0 1; do echo "rep $rep np $np"; TP_GEMM_WIDE_NP=$np timeout 300 python tools/gemm_bench.py --shapes 16384x16384x16384 --ops NN,TN --iters 30 --no-cublas 2>&1 | grep shape | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['shape'], d['op'], d['tflops'])"; done; done
for np in 0 1; do TP_GEMM_WIDE_NP=$np ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm --csv python tools/ncu_shapes.py --only c3h_fwd 2>/dev/null | grep -E "dram__bytes|duration|per_second" | awk -F'","' -v r=$np '{print "np" r, $(NF-2), $NF}'; done
python -m pytest tests/test_gpu_nccl.py -q -k "check_and_abort" 2>&1 | tail -2
python bench.py --no-cpu-baseline --no-e2e > /dev/null 2>&1; ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_c3head.csv python bench.py --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline > gpurun_out/ncu_c3head_bench.log 2>&1; echo "ncu launches rc=$?"
