"""One pre-LN Transformer block (TPBlock: LN, QKV, attention, proj, LN, fc1+GeLU, fc2, two
residuals) forward + backward on one GPU through the C ABI, CUDA-graph replay.

    python tools/transformer_bench.py [--workload c5] [--steps 5]

C5 (GPT): batch 8 x seq 2048 tokens, h = 8192, 64 heads, F = 32768.
Reports TFLOP/s of the block's GEMM + attention flops and the phase shares of one eager step.
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402
from paper_2110_14883_b200.block import TPBlock  # noqa: E402

WL = {"c5": dict(seq=2048, batch=8, h=8192, heads=64, F=32768),
      "c5-small": dict(seq=2048, batch=2, h=4096, heads=32, F=16384)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5", choices=sorted(WL))
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    w = WL[a.workload]
    M = w["seq"] * w["batch"]
    g = api.tp_grid_init("1d", 1, 0)
    blk = TPBlock(g, M, w["h"], w["heads"], w["seq"], F=w["F"])
    blk.fill()
    for _ in range(2):
        blk.step()
    torch.cuda.synchronize()
    # phase shares (eager, one step)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    blk.forward()
    ev[1].record()
    blk.backward()
    ev[2].record()
    torch.cuda.synchronize()
    fwd_ms, bwd_ms = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        blk.step()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        gr.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(json.dumps({"workload": a.workload, "block": "pre-LN transformer block fwd+bwd, 1 GPU",
                      "M": M, **w, "ms_per_step": round(ms, 3),
                      "tflops": round(blk.flops() / ms / 1e9, 1),
                      "eager_fwd_ms": round(fwd_ms, 3), "eager_bwd_ms": round(bwd_ms, 3)}))


if __name__ == "__main__":
    main()
