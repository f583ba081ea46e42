"""Ring Self-Attention forward on one GPU (ring of 1: the local work of every rank), CUDA
events. Reports ms, attention TFLOP/s (4 s^2 d per head: QK^T + PV) and the achieved HBM
bandwidth of the score round trip the paper's two-pass algorithm implies per head:
write S (fp32) + read S + write P (2 B) + read P = 12 B per score."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402


def main():
    s, d, heads = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (8192, 64, 16)))
    g = api.tp_grid_init("1d", 1, 0)
    ds = api.rsa_desc(s, d, heads, "bf16")
    q, k, v = (torch.randn(heads, s, d, device="cuda").to(torch.bfloat16) for _ in range(3))
    out = torch.empty_like(q)
    ws = torch.empty(api.tp_rsa_ws_size(g, ds), device="cuda", dtype=torch.uint8)
    run = lambda: api.tp_rsa_fwd(g, ds, q, k, v, out, ws)
    for _ in range(3):
        run()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        run()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 5
    e0.record()
    for _ in range(n):
        gr.replay()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / n
    flops = 4.0 * s * s * d * heads
    score_bytes = 12.0 * s * s * heads
    ref = torch.nn.functional.scaled_dot_product_attention(q[None].float(), k[None].float(), v[None].float())[0]
    err = float((out.float() - ref).norm() / ref.norm())
    # backward: the fused ring backward (lse from the forward) vs the two-pass form
    lse = torch.empty(heads * s, device="cuda", dtype=torch.float32)
    api.tp_rsa_fwd(g, ds, q, k, v, out, ws, lse=lse)
    do = torch.randn_like(q)
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)

    def t_of(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps

    fused = t_of(lambda: api.tp_rsa_bwd(g, ds, q, k, v, do, dq, dk, dv, ws, out=out, lse=lse))
    two = t_of(lambda: api.tp_rsa_bwd(g, ds, q, k, v, do, dq, dk, dv, ws))
    print(json.dumps({"op": "rsa_fwd", "s": s, "d_k": d, "heads": heads, "ms": round(ms, 4),
                      "tflops": round(flops / ms / 1e9, 1),
                      "score_roundtrip_gbs": round(score_bytes / ms / 1e6, 1),
                      "rel_err_vs_torch_sdpa_fp32": round(err, 5),
                      "bwd_fused_ms": round(fused, 4), "bwd_fused_tflops": round(2.5 * flops / fused / 1e9, 1),
                      "bwd_two_pass_ms": round(two, 4), "bwd_two_pass_tflops": round(2.5 * flops / two / 1e9, 1)}))


if __name__ == "__main__":
    main()
