"""Diagnostic: cuBLAS (torch.matmul) and tp_gemm on the C2 forward shape 512 x 4096 x 4096
(and the backward's NT / TN products) for a side-by-side ncu capture."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_14883_b200 import api  # noqa: E402

M, K, N = 512, 4096, 4096
A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
B = torch.randn(K, N, device="cuda").to(torch.bfloat16)
ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
for _ in range(3):
    C = torch.matmul(A, B)
    D = torch.empty_like(C)
    api.tp_gemm(0, 0, M, N, K, "bf16", A, K, B, N, None, 0, D, N, "bf16", 1.0, None, None, ws)
torch.cuda.synchronize()
print("max diff", (C.float() - D.float()).abs().max().item())
