for w in c2 c3 c4 c5 c3head; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/r02_bench_$w.json 2>gpurun_out/r02_bench_$w.err; python -c "
import json; d=json.load(open('gpurun_out/r02_bench_$w.json'))
r=d['roofline']; print('$w', d['value'], d['ms_per_step'], r['bound'], r['achieved'], r['unit'], r['frac'], d['e2e']['value'], d['clocks']['sm_mhz'])"; done
