mkdir -p gpurun_out/san
ncu --set full --clock-control none --import-source on -k regex:gemm -o gpurun_out/ncu_shapes python tools/ncu_shapes.py > gpurun_out/ncu_shapes.log 2>&1
echo "ncu rc=$?"
for tool in memcheck racecheck synccheck; do
  for c in owner exchange ragged; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_gemm.py --case $c > gpurun_out/san/${tool}_$c.log 2>&1; echo "$tool $c rc=$?"
  done
  TP_GEMM_SPLIT_OWNER=0 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_gemm.py --case lastarriver > gpurun_out/san/${tool}_lastarriver.log 2>&1; echo "$tool lastarriver rc=$?"
  TP_GEMM_MC=5 timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_gemm.py --case mc5 > gpurun_out/san/${tool}_mc5.log 2>&1; echo "$tool mc5 rc=$?"
done
tail -3 gpurun_out/san/*.log | head -80
