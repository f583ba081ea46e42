for rep in 1 2 3; do for w in 0 1; do echo "rep $rep wide $w"; TP_GEMM_WIDE=$w timeout 300 python tools/gemm_bench.py --shapes 16384x16384x16384,8192x8192x8192,8192x16384x4096,16384x4096x8192 --ops NN,NT,TN --iters 30 --no-cublas 2>&1 | grep shape | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['shape'], d['op'], d['tflops'])"; done; done
