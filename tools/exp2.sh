S=512x4096x4096
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,launch__grid_size,launch__cluster_dim_x,launch__block_size,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python tools/gemm_bench.py --shapes $S,4096x4096x512 --ops NN --iters 2 > gpurun_out/exp2_auto.csv 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,launch__grid_size,launch__cluster_dim_x,launch__block_size,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python tools/gemm_bench.py --shapes $S --ops NN --iters 2 --no-split --no-cublas > gpurun_out/exp2_nosplit.csv 2>&1
TP_GEMM_KERNEL=1 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,launch__grid_size,launch__cluster_dim_x,lts__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv python tools/gemm_bench.py --shapes $S --ops NN --iters 2 --no-cublas > gpurun_out/exp2_v1.csv 2>&1
python - <<'PY'
import time, torch, sys
sys.path.insert(0,'.')
from paper_2110_14883_b200 import api
M,N,K=512,4096,4096
A=torch.randn(M,K,device='cuda').bfloat16(); B=torch.randn(K,N,device='cuda').bfloat16(); D=torch.empty(M,N,device='cuda').bfloat16()
ws=torch.empty(api.tp_gemm_ws_bytes(),device='cuda',dtype=torch.uint8)
for _ in range(5): api.tp_gemm(0,0,M,N,K,'bf16',A,K,B,N,None,N,D,N,'bf16',ws=ws)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(200): api.tp_gemm(0,0,M,N,K,'bf16',A,K,B,N,None,N,D,N,'bf16',ws=ws)
t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
print('host us per tp_gemm call', (t1-t)/200*1e6, 'total incl gpu', (t2-t)/200*1e6)
g=api.tp_grid_init('1d',1,0); d=api.desc(M,K,N)
wsb,_=api.tp_workspace_size(g,d); w2=torch.empty(wsb,device='cuda',dtype=torch.uint8)
X=A; W=B; Y=D
for _ in range(5): api.tp_linear_fwd(g,d,X,W,None,Y,None,w2)
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(200): api.tp_linear_fwd(g,d,X,W,None,Y,None,w2)
t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
print('host us per tp_linear_fwd call', (t1-t)/200*1e6, 'total incl gpu', (t2-t)/200*1e6)
PY
