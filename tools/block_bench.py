"""Transformer MLP block through the C ABI on one GPU (NEXT-2 measurement): LayerNorm ->
fc1 (+ GeLU) -> fc2, forward + backward, CUDA-graph replay, CUDA events.

    python tools/block_bench.py [--workload c5|c4] [--steps 10]

C5 (GPT): M = 8 x 2048 tokens, h = 8192, fc1 8192 -> 32768, fc2 32768 -> 8192.
C4 (ViT-S/16): M = 4096 x 197 tokens, h = 384, fc1 384 -> 1536, fc2 1536 -> 384.
Reports block TFLOP/s (GEMM flops only: 6 M h F per linear pair x 2) and the time shares of
the LayerNorm, GeLU and GEMM kernels (per-kernel events of one instrumented eager step).
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402

WL = {"c5": (8 * 2048, 8192, 32768), "c4": (4096 * 197, 384, 1536)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5", choices=sorted(WL))
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    M, h, F = WL[a.workload]
    g = api.tp_grid_init("1d", 1, 0)
    bf = torch.bfloat16
    d1 = api.desc(M, h, F, "bf16", split_1d=0, flags=api.TP_FLAG_GELU)
    d2 = api.desc(M, F, h, "bf16", split_1d=1)
    dn = api.desc(M, h, F, "bf16")  # LayerNorm input = fc1's X layout
    x = torch.randn(M, h, device="cuda").to(bf)
    ln_y = torch.empty_like(x)
    gam = torch.ones(h, device="cuda", dtype=bf)
    bet = torch.zeros(h, device="cuda", dtype=bf)
    stats = torch.empty(M, 2, device="cuda")
    W1 = (torch.randn(h, F, device="cuda") * 0.02).to(bf)
    W2 = (torch.randn(F, h, device="cuda") * 0.02).to(bf)
    b1 = torch.zeros(F, device="cuda", dtype=bf)
    H1 = torch.empty(M, F, device="cuda", dtype=bf)
    Y = torch.empty(M, h, device="cuda", dtype=bf)
    dY = torch.randn(M, h, device="cuda").to(bf)
    dH1 = torch.empty_like(H1)
    dLN = torch.empty_like(x)
    dX = torch.empty_like(x)
    dW1, dW2 = torch.empty_like(W1), torch.empty_like(W2)
    db1 = torch.empty_like(b1)
    dg, dbt = torch.empty_like(gam), torch.empty_like(bet)
    s1 = api.tp_workspace_size(g, d1)
    s2 = api.tp_workspace_size(g, d2)
    ws = torch.empty(max(s1[0], s2[0], api.tp_layernorm_ws_size(g, dn, "X")), device="cuda",
                     dtype=torch.uint8)
    sv1 = torch.empty(s1[1], device="cuda", dtype=torch.uint8)
    sv2 = torch.empty(max(s2[1], 1), device="cuda", dtype=torch.uint8) if s2[1] else None

    def step(ev=None):
        mark = (lambda n: ev.append((n, torch.cuda.Event(enable_timing=True)))) if ev is not None else (lambda n: None)

        def rec(n):
            mark(n)
            if ev is not None:
                ev[-1][1].record()
        rec("start")
        api.tp_layernorm_fwd(g, dn, "X", 1e-5, x, gam, bet, ln_y, stats, ws)
        rec("ln_fwd")
        api.tp_linear_fwd(g, d1, ln_y, W1, b1, H1, sv1, ws)
        rec("fc1_fwd+gelu")
        api.tp_linear_fwd(g, d2, H1, W2, None, Y, sv2, ws)
        rec("fc2_fwd")
        api.tp_linear_bwd(g, d2, dY, H1, W2, sv2, dH1, dW2, None, ws)
        rec("fc2_bwd")
        api.tp_linear_bwd(g, d1, dH1, ln_y, W1, sv1, dLN, dW1, db1, ws)
        rec("fc1_bwd+gelu")
        api.tp_layernorm_bwd(g, dn, "X", dLN, x, gam, stats, dX, dg, dbt, ws)
        rec("ln_bwd")

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = []
    step(ev)
    torch.cuda.synchronize()
    shares = {ev[i][0]: round(ev[i - 1][1].elapsed_time(ev[i][1]), 4) for i in range(1, len(ev))}
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        step()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        gr.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    flops = 2 * 6.0 * M * h * F
    print(json.dumps({"workload": a.workload, "block": "LN -> fc1+GeLU -> fc2, fwd+bwd, 1 GPU",
                      "M": M, "h": h, "F": F, "ms_per_step": round(ms, 4),
                      "tflops_gemm_flops": round(flops / ms / 1e9, 1), "eager_ms_by_phase": shares}))


if __name__ == "__main__":
    main()
