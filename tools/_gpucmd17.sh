for rep in 1 2; do for r in 8 4 2 16; do echo "rep $rep raster $r"; TP_GEMM_WIDE_RASTER=$r timeout 300 python tools/gemm_bench.py --shapes 16384x16384x16384 --ops NN,TN --iters 30 --no-cublas 2>&1 | grep shape | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['shape'], d['op'], d['tflops'])"; done; done
for r in 8 4 2; do TP_GEMM_WIDE_RASTER=$r ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm --csv python tools/ncu_shapes.py --only c3h_fwd 2>/dev/null | grep -E "dram__bytes|duration|per_second" | awk -F'","' -v r=$r '{print "r" r, $(NF-2), $NF}'; done
