"""Where does the CTA-pair GEMM spend its cycles?  Runs one tp_gemm with the clock64 trace on
and prints per-role wait fractions (averaged over CTAs).

    python tools/gemm_trace.py 512x4096x4096 NN
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402

OPS = {"NN": (0, 0), "NT": (0, 1), "TN": (1, 0), "TT": (1, 1)}


def main():
    shp = sys.argv[1] if len(sys.argv) > 1 else "512x4096x4096"
    op = sys.argv[2] if len(sys.argv) > 2 else "NN"
    M, N, K = map(int, shp.split("x"))
    ta, tb = OPS[op]
    data = next((a.split("=")[1] for a in sys.argv if a.startswith("--data=")), "randn")
    gen = {"randn": torch.randn, "zeros": torch.zeros, "ones": torch.ones,
           "uniform": lambda *s, **k: torch.rand(*s, **k) * 2 - 1,
           "ternary": lambda *s, **k: torch.randint(-1, 2, s, **k).float()}[data]
    A = gen(*((K, M) if ta else (M, K)), device="cuda").to(torch.bfloat16)
    B = gen(*((N, K) if tb else (K, N)), device="cuda").to(torch.bfloat16)
    D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    tr = torch.zeros(300 * 16, device="cuda", dtype=torch.int64)
    run = lambda: api.tp_gemm(ta, tb, M, N, K, "bf16", A, A.shape[1], B, B.shape[1], None, N, D, N,
                              "bf16", ws=ws)
    hot = "--hot" in sys.argv
    run()
    api.tp_gemm_trace(tr)
    if not hot:
        api.tp_l2_flush(flush)
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    api.tp_gemm_trace(None)
    t = tr.view(-1, 16).cpu().double()
    live = t[:, 1] > 0
    t = t[live]
    names = ["prod_wait_empty", "prod_total", "mma_wait_full", "mma_wait_tmem", "mma_total",
             "epi_wait_tfull", "epi_total"]
    out = {"shape": shp, "op": op, "ctas": int(live.sum())}
    for i, n in enumerate(names):
        col = t[:, i]
        nz = col[col > 0] if i in (2, 3, 4) else col
        out[n] = round(float(nz.mean()), 0) if len(nz) else 0
    ent, pro, ext = t[:, 7], t[:, 8], t[:, 9]
    out["event_us"] = round(e0.elapsed_time(e1) * 1000, 2)
    out["span_us"] = round(float(ext.max() - ent.min()) / 1000, 2)
    out["entry_spread_us"] = round(float(ent.max() - ent.min()) / 1000, 2)
    out["prologue_us"] = round(float((pro - ent).mean()) / 1000, 2)
    out["cta_us"] = round(float((ext - ent).mean()) / 1000, 2)
    out["exit_spread_us"] = round(float(ext.max() - ext.min()) / 1000, 2)
    out["sm_mhz"] = round(float(((t[:, 11] - t[:, 10]) / (ext - ent)).mean()) * 1000, 0)
    first = t[:, 12][t[:, 12] > 0]
    out["mma_wait_first_kb"] = round(float(first.mean()), 0) if len(first) else 0
    st, ns = t[:, 13], t[:, 14]
    out["steady_cyc_per_kb"] = round(float(st.sum() / max(ns.sum(), 1)), 1)
    xw = t[:, 15].long()
    out["epi_split_publish"] = round(float((xw & 0xffffffff).double().mean()), 0)
    out["epi_split_wait"] = round(float((xw >> 32).double().mean()), 0)
    out["mma_full_wait_frac"] = round(out["mma_wait_full"] / max(out["mma_total"], 1), 3)
    out["prod_wait_frac"] = round(out["prod_wait_empty"] / max(out["prod_total"], 1), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
