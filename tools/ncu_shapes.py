"""Launch every distinct local-GEMM shape of SURVEY 8(d) once through tp_gemm (the kernel the
schedules call), for an ncu capture of each (tools/ncu_summary.py reads the report).

    ncu --set full --clock-control none --import-source on -k regex:gemm \
        -o gpurun_out/ncu_shapes python tools/ncu_shapes.py [--only NAME ...]

Shapes (m x k x n, per rank; "NN" = X.W, "NT" = dY.W^T (dX), "TN" = X^T.dY (dW)):
  c2_fwd        512 x 4096 x 4096 NN        C2, 1D p=1 forward (bench N=1 before round 2)
  c3h_fwd       16384^3 NN                  C3-HEAD p=1 forward (bench N=1 headline)
  c3h_dx/dw     16384^3 NT / TN             C3-HEAD p=1 backward
  c3h_2d_*      8192^3 NN / NT / TN         C3-HEAD 2D q=2 and 3D l=2 per-rank products
  c3h_25d       4096 x 8192 x 8192 NN       C3-HEAD 2.5D q=2 d=2 per-rank SUMMA step
  c3h_1d8       16384 x 16384 x 2048 NN     C3-HEAD 1D p=8 column-split forward
  c4_dw         192 x 403456 x 576 TN       C4 ViT-S QKV dW, 2D q=2 (long K: split-K)
  c5_fc1        8192 x 4096 x 16384 NN      C5 GPT fc1 forward, 3D l=2
  c5_fc2_dw     16384 x 8192 x 4096 TN      C5 GPT fc2 dW, 3D l=2
Inputs: the library's seeded generator (tp_fill), bf16, fp32 accumulate, bf16 out.
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2110_14883_b200 import api  # noqa: E402

SHAPES = {  # name: (M, K, N, trans_a, trans_b)
    "c2_fwd": (512, 4096, 4096, 0, 0),
    "c3h_fwd": (16384, 16384, 16384, 0, 0),
    "c3h_dx": (16384, 16384, 16384, 0, 1),
    "c3h_dw": (16384, 16384, 16384, 1, 0),
    "c3h_2d_nn": (8192, 8192, 8192, 0, 0),
    "c3h_2d_nt": (8192, 8192, 8192, 0, 1),
    "c3h_2d_tn": (8192, 8192, 8192, 1, 0),
    "c3h_25d": (4096, 8192, 8192, 0, 0),
    "c3h_1d8": (16384, 16384, 2048, 0, 0),
    "c4_dw": (192, 403456, 576, 1, 0),
    "c5_fc1": (8192, 4096, 16384, 0, 0),
    "c5_fc2_dw": (16384, 8192, 4096, 1, 0),
}


def operand(rows, cols, tid):
    t = torch.empty(rows, cols, device="cuda", dtype=torch.bfloat16)
    api.tp_fill(t, "bf16", rows, cols, cols, 42, tid, "uniform", 1.0, 0, 0, cols)
    return t


def run(name, reps):
    M, K, N, ta, tb = SHAPES[name]
    A = operand(K, M, 1) if ta else operand(M, K, 1)
    B = operand(N, K, 2) if tb else operand(K, N, 2)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    lda, ldb = (M if ta else K), (K if tb else N)
    for _ in range(reps):
        api.tp_gemm(ta, tb, M, N, K, "bf16", A, lda, B, ldb, None, 0, D, N, "bf16", 1.0, None,
                    None, ws)
    torch.cuda.synchronize()
    print(f"{name}: M={M} K={K} N={N} ta={ta} tb={tb} flops={2.0 * M * N * K:.4e}", flush=True)
    del A, B, D, ws
    torch.cuda.empty_cache()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--reps", type=int, default=1)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    for name in (a.only or SHAPES):
        run(name, a.reps)


if __name__ == "__main__":
    main()
