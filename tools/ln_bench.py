"""LayerNorm fwd / bwd timing on one GPU (p = 1: no reductions), achieved GB/s of the
algorithmic bytes (fwd: read x + write y; bwd: read dy, x + write dx; bf16), CUDA events."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402


def main():
    M, H = (int(v) for v in (sys.argv[1:3] if len(sys.argv) > 2 else (16384, 8192)))
    g = api.tp_grid_init("1d", 1, 0)
    ds = api.desc(M, H, H, "bf16")
    x = torch.randn(M, H, device="cuda").to(torch.bfloat16)
    dy = torch.randn(M, H, device="cuda").to(torch.bfloat16)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    gam = torch.ones(H, device="cuda", dtype=torch.bfloat16)
    bet = torch.zeros(H, device="cuda", dtype=torch.bfloat16)
    dg, db = torch.empty_like(gam), torch.empty_like(bet)
    st = torch.empty(M, 2, device="cuda")
    ws = torch.empty(api.tp_layernorm_ws_size(g, ds, "X"), device="cuda", dtype=torch.uint8)
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    fwd = lambda: api.tp_layernorm_fwd(g, ds, "X", 1e-5, x, gam, bet, y, st, ws)
    bwd = lambda: api.tp_layernorm_bwd(g, ds, "X", dy, x, gam, st, dx, dg, db, ws)
    for name, fn, nbytes in (("fwd", fwd, 2 * M * H * 2), ("bwd", bwd, 3 * M * H * 2)):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(10):
            api.tp_l2_flush(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sorted(ts)[len(ts) // 2]
        print(json.dumps({"op": f"layernorm_{name}", "M": M, "H": H, "ms": round(ms, 4),
                          "alg_bytes": nbytes, "gbs": round(nbytes / ms / 1e6, 1)}))


if __name__ == "__main__":
    main()
