"""Micro-benchmark of the library's local GEMM (tp_gemm) on one GPU, CUDA-event timed.

    python tools/gemm_bench.py [--shapes 8192x8192x8192,512x4096x4096] [--ops NN,NT,TN] [--iters 20]
Set TP_GEMM_KERNEL=1 to force the 1-CTA kernel. Prints one JSON line per (shape, op).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402

OPS = {"NN": (0, 0), "NT": (0, 1), "TN": (1, 0), "TT": (1, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default="512x4096x4096,4096x4096x512,8192x8192x8192")
    ap.add_argument("--ops", default="NN,NT,TN")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--no-split", action="store_true")
    ap.add_argument("--out", default="bf16")
    ap.add_argument("--no-flush", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--hot-graph", action="store_true")
    a = ap.parse_args()
    ws = None if a.no_split else torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    for shp in a.shapes.split(","):
        M, N, K = map(int, shp.split("x"))
        for op in a.ops.split(","):
            ta, tb = OPS[op]
            A = torch.randn((K, M) if ta else (M, K), device="cuda").to(torch.bfloat16)
            B = torch.randn((N, K) if tb else (K, N), device="cuda").to(torch.bfloat16)
            D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16 if a.out == "bf16" else torch.float32)
            lda, ldb = A.shape[1], B.shape[1]
            run = lambda: api.tp_gemm(ta, tb, M, N, K, "bf16", A, lda, B, ldb, None, N, D, N, a.out,
                                      ws=ws)
            for _ in range(3):
                run()
            ts = []
            for _ in range(a.iters):
                if not a.no_flush:
                    api.tp_l2_flush(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ts.sort()
            med = ts[len(ts) // 2]
            if a.hot_graph:   # back-to-back launches in one graph, operands L2-resident
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    for _ in range(10):
                        run()
                gr.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gr.replay()
                e1.record()
                e1.synchronize()
                med = e0.elapsed_time(e1) / 10
            # reference: torch.matmul (cuBLAS) for context
            At = A.t() if ta else A
            Bt = B.t() if tb else B
            for _ in range(3):
                torch.matmul(At, Bt)
            tc = [med]
            for _ in range(0 if a.no_cublas else a.iters):
                api.tp_l2_flush(flush)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                torch.matmul(At, Bt)
                e1.record()
                e1.synchronize()
                tc.append(e0.elapsed_time(e1))
            tc.sort()
            if a.hot_graph and not a.no_cublas:
                gr2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr2):
                    for _ in range(10):
                        torch.matmul(At, Bt)
                gr2.replay()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gr2.replay()
                e1.record()
                e1.synchronize()
                tc = [e0.elapsed_time(e1) / 10]
            flops = 2.0 * M * N * K
            print(json.dumps({"shape": shp, "op": op, "kernel": os.environ.get("TP_GEMM_KERNEL", "auto"), "pf": os.environ.get("TP_GEMM_PREFETCH", "0"), "split": not a.no_split, "flush": not a.no_flush,
                              "ms": round(med, 4), "tflops": round(flops / med / 1e9, 1),
                              "cublas_ms": round(tc[len(tc) // 2], 4),
                              "cublas_tflops": round(flops / tc[len(tc) // 2] / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
