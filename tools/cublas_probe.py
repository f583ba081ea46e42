"""Diagnostic: one torch.matmul (cuBLAS) and one tp_gemm launch of the same bf16 shape, for a
side-by-side ncu capture (power-capped efficiency comparison of the 16384^3 product)."""
import sys
import os
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_14883_b200 import api  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
A = torch.randn(n, n, device="cuda").to(torch.bfloat16)
B = torch.randn(n, n, device="cuda").to(torch.bfloat16)
C = torch.matmul(A, B)
D = torch.empty_like(C)
ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
api.tp_gemm(0, 0, n, n, n, "bf16", A, n, B, n, None, 0, D, n, "bf16", 1.0, None, None, ws)
torch.cuda.synchronize()
print("max diff", (C.float() - D.float()).abs().max().item())
