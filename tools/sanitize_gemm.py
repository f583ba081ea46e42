"""compute-sanitizer targets: small GEMMs through the cross-CTA protocols of the pair kernel,
checked against torch after the run (the sanitizer reports races / sync errors / bad accesses).

    compute-sanitizer --tool racecheck  python tools/sanitize_gemm.py
    compute-sanitizer --tool synccheck  python tools/sanitize_gemm.py
    compute-sanitizer --tool memcheck   python tools/sanitize_gemm.py
    TP_GEMM_MC=5 compute-sanitizer ... python tools/sanitize_gemm.py --case mc5

Cases: split-K with split 0 keeping its tile in TMEM and waiting for its sibling (owner-wait),
the two-split reduce-scatter exchange, the last-arriver reduction (owner-wait off), the grouped
dX + dW launch, and the DSMEM K-split cluster (TP_GEMM_MC=5).
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_14883_b200 import api  # noqa: E402

CASES = {  # name: list of (M, K, N, ta, tb)
    "owner": [(256, 4096, 256, 0, 0)],          # 1 pair tile, long K: split many ways
    "exchange": [(512, 1024, 4096, 0, 0)],      # 32 pair tiles: two splits, exchange path
    "lastarriver": [(256, 2048, 512, 1, 0)],
    "mc5": [(512, 1024, 1024, 0, 0)],
    "ragged": [(300, 520, 200, 0, 1)],
}


def check(M, K, N, ta, tb):
    g = torch.Generator(device="cuda").manual_seed(M + K + N)
    A = torch.randn((K, M) if ta else (M, K), device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn((N, K) if tb else (K, N), device="cuda", generator=g).to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.float32)
    ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    api.tp_gemm(ta, tb, M, N, K, "bf16", A, M if ta else K, B, K if tb else N, None, 0, D, N,
                "fp32", 1.0, None, None, ws)
    torch.cuda.synchronize()
    ref = (A.t() if ta else A).double() @ (B.t() if tb else B).double()
    err = ((D.double() - ref).norm() / ref.norm()).item()
    print(f"M={M} K={K} N={N} ta={ta} tb={tb}: rel {err:.2e}", flush=True)
    assert err < 1e-5


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", nargs="*", default=["owner", "exchange", "ragged"])
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for c in a.case:  # "lastarriver" runs with TP_GEMM_SPLIT_OWNER=0, "mc5" with TP_GEMM_MC=5
        for shape in CASES[c]:
            print(c, end=" ")
            check(*shape)


if __name__ == "__main__":
    main()
