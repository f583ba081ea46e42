# round-end style verification: smoke, full GPU suite, bench lines for every workload, the C2 ncu launch list
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gputests_full.log 2>&1; echo tests=$?; tail -2 gpurun_out/gputests_full.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu_c2.csv python bench.py --steps 2 --warmup 3 --eager --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/ncu_c2.csv c2 1 > gpurun_out/ncu_c2_summary.txt 2>&1
python bench.py > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err
for w in c3head c5 c4 c3; do python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/bench_$w.json 2>gpurun_out/bench_$w.err; done
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2>&1
for f in gpurun_out/bench_*.json; do echo $f; cut -c1-400 $f; done
