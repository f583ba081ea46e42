"""Probe: tcgen05 GEMM on the ragged attention-backward shapes (b = 197 rows, padded row
strides) against a float64 torch reference. Diagnostic only."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2110_14883_b200 import api

torch.manual_seed(0)
def run(M, N, K, ta, tb, lda, ldb, ws=True):
    A = torch.randn((K, lda) if ta else (M, lda), device="cuda").to(torch.bfloat16)
    B = torch.randn((N, ldb) if tb else (K, ldb), device="cuda").to(torch.bfloat16)
    Ae = (A[:, :M].t() if ta else A[:, :K]).double()
    Be = (B[:, :K].t() if tb else B[:, :N]).double()
    ref = Ae @ Be
    D = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float32)
    w = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8) if ws else None
    api.tp_gemm(ta, tb, M, N, K, "bf16", A, lda, B, ldb, None, 0, D, N, "fp32", 1.0, None, None, w)
    torch.cuda.synchronize()
    err = ((D.double() - ref).norm() / ref.norm()).item()
    print(f"M={M} N={N} K={K} ta={ta} tb={tb} lda={lda} ldb={ldb} ws={ws}: rel {err:.2e} "
          f"nan={torch.isnan(D).sum().item()}")

for ws in (True, False):
    run(197, 64, 197, 0, 0, 200, 64, ws)    # dQ = dS K
    run(197, 64, 197, 1, 0, 200, 64, ws)    # dK parts = dS^T Q
    run(197, 197, 64, 0, 1, 64, 64, ws)     # S = Q K^T
    run(512, 64, 512, 0, 0, 512, 64, ws)
    run(130, 64, 130, 0, 0, 136, 64, ws)
    run(197, 64, 197, 0, 0, 200, 64, ws)
    run(300, 64, 197, 0, 0, 200, 64, ws)
    run(197, 64, 256, 0, 0, 256, 64, ws)
    run(256, 64, 197, 0, 0, 200, 64, ws)

import os
print(os.environ.get("TP_GEMM_KERNEL"), os.environ.get("TP_GEMM_V1_TMA_STORE"))
print("--- padded ldd: padding columns must stay untouched")
def run_pad(M, N, K, ldd, out="fp32", tb=1):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn((N, K) if tb else (K, N), device="cuda").to(torch.bfloat16)
    ref = A.double() @ (B.double().t() if tb else B.double())
    dt = torch.float32 if out == "fp32" else torch.bfloat16
    D = torch.full((M, ldd), float("-inf"), device="cuda", dtype=dt)
    w = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    api.tp_gemm(0, tb, M, N, K, "bf16", A, K, B, K if tb else N, None, 0, D, ldd, out, 1.0, None, None, w)
    torch.cuda.synchronize()
    err = ((D[:, :N].double() - ref).norm() / ref.norm()).item()
    pad = D[:, N:]
    bad = ~torch.isinf(pad)
    pad_ok = not bool(bad.any().item())
    info = ""
    if not pad_ok:
        idx = bad.nonzero()
        info = (f" clobbered={int(bad.sum())} rows {idx[:,0].min().item()}..{idx[:,0].max().item()}"
                f" cols {N + idx[:,1].min().item()}..{N + idx[:,1].max().item()} sample={pad[bad][:4].tolist()}")
    print(f"M={M} N={N} K={K} ldd={ldd} out={out}: rel {err:.2e} pad untouched={pad_ok}{info}")
run_pad(197, 197, 64, 200)
run_pad(197, 197, 64, 200, "bf16")
run_pad(130, 130, 64, 136)
run_pad(512, 512, 64, 512)
pass
