for dh in 64 128; do for seq in 128 200 256 384 1024; do for B in 1 2; do
timeout 30 python -c "
import sys, numpy as np, torch
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import synth
from test_gpu_flash import run_core
from paper_2110_14883_b200 import api
from oracle import mha
from tp_harness import rel_fro
B,seq,heads,dh=$B,$seq,3,$dh
q=synth.tensor(41,0,B*seq,3*heads*dh,dtype='bf16').astype(np.float64)*2
got=run_core(api,B,seq,heads,dh,q)
print('dh',dh,'seq',seq,'B',B,'err',rel_fro(got,mha.mha_fwd(q,seq,heads)))
" 2>&1 | tail -1 || echo "dh $dh seq $seq B $B TIMEOUT/FAIL"
done; done; done
