"""Attention core forward / backward timing on one GPU (tp_attention_fwd / _bwd, 1D p=1): the
fused backward (lse from the forward, flash_bwd.cu) against the two-pass backward (scores
recomputed through HBM).

    python tools/attn_bench.py [--seq 2048 --batch 8 --heads 64 --dh 128] [--iters 10]

Flops: forward 4 s^2 d per (sequence, head); backward 8 s^2 d (4 products) + the recomputed QK^T
(2 s^2 d) = 10 s^2 d (FlashAttention's accounting: 2.5x the forward).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=2048)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--heads", type=int, default=64)
    ap.add_argument("--dh", type=int, default=128)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    h = a.heads * a.dh
    M = a.seq * a.batch
    g = api.tp_grid_init("1d", 1, 0)
    dq = api.desc(M, h, 3 * h)
    qkv = (torch.randn(M, 3 * h, device="cuda") * 0.5).to(torch.bfloat16)
    out = torch.empty(M, h, device="cuda", dtype=torch.bfloat16)
    dout = torch.randn(M, h, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    lse = torch.empty(M * a.heads, device="cuda", dtype=torch.float32)
    ws = torch.empty(api.tp_attention_ws_size(g, dq, a.seq, a.heads), device="cuda", dtype=torch.uint8)

    def timeit(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / a.iters

    fwd = timeit(lambda: api.tp_attention_fwd(g, dq, a.seq, a.heads, qkv, out, ws, lse=lse))
    bwd_fused = timeit(lambda: api.tp_attention_bwd(g, dq, a.seq, a.heads, qkv, dout, dqkv, ws,
                                                    out=out, lse=lse))
    ref = dqkv.clone()
    bwd_two = timeit(lambda: api.tp_attention_bwd(g, dq, a.seq, a.heads, qkv, dout, dqkv, ws))
    diff = ((dqkv.float() - ref.float()).norm() / ref.float().norm()).item()
    core = a.batch * a.heads * a.seq * a.seq * a.dh
    print(json.dumps({"seq": a.seq, "batch": a.batch, "heads": a.heads, "dh": a.dh,
                      "fwd_ms": round(fwd, 3), "fwd_tflops": round(4 * core / fwd / 1e9, 1),
                      "bwd_fused_ms": round(bwd_fused, 3),
                      "bwd_fused_tflops": round(10 * core / bwd_fused / 1e9, 1),
                      "bwd_two_pass_ms": round(bwd_two, 3),
                      "bwd_two_pass_tflops": round(10 * core / bwd_two / 1e9, 1),
                      "rel_diff_fused_vs_two_pass": round(diff, 5)}))
    api.tp_grid_destroy(g)


if __name__ == "__main__":
    main()
