# Cluster-multicast variants on the 512-row GEMMs after the v3 issue-loop fix (hot graph)
S=512x4096x4096
for mc in 1 2 3 4; do
  echo "== pair BN=128 MC=$mc"
  TP_GEMM_KERNEL=2 TP_GEMM_BN=128 TP_GEMM_MC=$mc python tools/gemm_bench.py --shapes $S --ops NN,NT --hot-graph --no-cublas | cut -c1-110
  echo "== pair BN=256 MC=$mc"
  TP_GEMM_KERNEL=2 TP_GEMM_BN=256 TP_GEMM_MC=$mc python tools/gemm_bench.py --shapes $S --ops NN,NT --hot-graph --no-cublas | cut -c1-110
done
echo "== 1-CTA"; TP_GEMM_KERNEL=1 python tools/gemm_bench.py --shapes $S --ops NN,NT --hot-graph | cut -c1-200
