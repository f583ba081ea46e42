"""Analytic communication / roofline model of the tensor-parallel linear layer (SURVEY 8(d),
NEXT-4's "analytic comm-volume/scaling CLI"): for a workload of BASELINE.json's configs and
every grid the paper defines at the given GPU counts, print the paper's Table volume next to
the volume this library's schedule moves, per-GPU NVLink bytes, per-GPU flops, the tensor and
link times and which one bounds the step. Host only; the numbers come from tp_cost_model
(libtp_b200.so) — no device work.

    python -m paper_2110_14883_b200.costmodel [--workload c2] [--gpus 1,2,4,8] [--json]
"""
from __future__ import annotations

import argparse
import json
import os

from . import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKLOADS = {  # (M tokens, [(K, N) per linear layer]) -- BASELINE.json configs
    "c1": (16, [(64, 64), (64, 64)], "fp32"),
    "c2": (512, [(4096, 4096), (4096, 4096)], "bf16"),
    "c3": (64, [(16384, 16384), (16384, 16384)], "bf16"),
    "c3head": (16384, [(16384, 16384), (16384, 16384)], "bf16"),
    "c4": (4096 * 197, [(384, 1152), (384, 384), (384, 1536), (1536, 384)], "bf16"),
    "c5": (16384, [(8192, 24576), (8192, 8192), (8192, 32768), (32768, 8192)], "bf16"),
}


def grids(p):
    """The grids the paper defines at p GPUs: (label, mode, q, d)."""
    out = [("1d", "1d", 0, 1)]
    for q in range(1, 64):
        if q * q == p:
            out.append(("2d", "2d", q, 1))
        for d in range(1, p + 1):
            if d * q * q == p and q > 1:
                out.append((f"2.5d(d={d})", "2.5d", q, d))
                if d > 1 and q % d == 0:  # Solomonik's 2.5D (TP_FLAG_SOLOMONIK, reading N5)
                    out.append((f"2.5d-solomonik(d={d})", "2.5d", q, d))
        if q ** 3 == p:
            out.append(("3d", "3d", q, 1))
    return out


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["bf16_tflops"]), "measured"
    except (OSError, KeyError, ValueError):
        return 1590.0, "fallback"


def model(workload, p, link_gbs=900.0, peak_tflops=None):
    M, layers, dtype = WORKLOADS[workload]
    peak = peak_tflops if peak_tflops is not None else peaks()[0]
    rows = []
    for label, mode, q, d in grids(p):
        tot = {k: 0.0 for k in ("paper_elems", "counted_elems", "link_bytes", "flops",
                                "t_tensor_us", "t_link_us", "t_exposed_us")}
        ok = True
        for i, (K, N) in enumerate(layers):
            fl = api.TP_FLAG_SOLOMONIK if "solomonik" in label else 0
            ds = api.desc(M, K, N, dtype, split_1d=i % 2, parity_3d=i % 2, flags=fl)
            try:
                c = api.tp_cost_model(mode, p, ds, q=q, depth=d, peak_tflops=peak,
                                      link_gbs=link_gbs)
            except api.TPError:
                ok = False
                break
            for k in tot:
                tot[k] += c[k]
        if not ok:
            continue
        bound = "tensor" if tot["t_tensor_us"] >= tot["t_link_us"] else "link"
        roof = max(tot["t_tensor_us"], tot["t_link_us"])
        rows.append({"workload": workload, "grid": label, "gpus": p,
                     "gflop_per_gpu": round(tot["flops"] / 1e9, 1),
                     "link_mb_per_gpu": round(tot["link_bytes"] / 1e6, 1),
                     "t_tensor_us": round(tot["t_tensor_us"], 1),
                     "t_link_us": round(tot["t_link_us"], 1), "bound": bound,
                     "exposed_comm_us": round(tot["t_exposed_us"], 1),
                     "step_estimate_us": round(tot["t_tensor_us"] + tot["t_exposed_us"], 1),
                     "max_pct_of_peak": round(100 * tot["t_tensor_us"] / roof, 1) if roof else None,
                     "paper_table_elems": tot["paper_elems"],
                     "schedule_elems": tot["counted_elems"]})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--link-gbs", type=float, default=900.0)
    ap.add_argument("--json", action="store_true")
    a = ap.parse_args()
    rows = [r for p in map(int, a.gpus.split(",")) for r in model(a.workload, p, a.link_gbs)]
    if a.json:
        for r in rows:
            print(json.dumps(r))
        return
    hdr = ["grid", "gpus", "gflop_per_gpu", "link_mb_per_gpu", "t_tensor_us", "t_link_us", "bound",
           "max_pct_of_peak", "exposed_comm_us", "step_estimate_us"]
    print(" | ".join(hdr))
    for r in rows:
        print(" | ".join(str(r[h]) for h in hdr))


if __name__ == "__main__":
    main()
