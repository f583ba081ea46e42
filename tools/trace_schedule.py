"""Span trace of one tensor-parallel layer fwd + bwd on in-process ranks (LOCAL transport, one
GPU): every GEMM launch and every line collective with its device start / end (tp_prof_spans),
per rank. Shows which collectives run under which GEMMs (the schedules' overlap, a-13).

    python tools/trace_schedule.py [--mode 3d] [--M 16384] [--h 16384] [--rank 0] [--json out]

With LOCAL transport the collectives are copy-engine copies and small fp32 sum kernels, and all
ranks share the GPU, so absolute times are not multi-GPU times; the ORDER and overlap of each
rank's own GEMMs and collectives is what the trace shows.
"""
import argparse
import json
import os
import sys
import threading

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2110_14883_b200 import api  # noqa: E402
from paper_2110_14883_b200.mlp import TPMLP  # noqa: E402

GRIDS = {"1d": (8, 1), "2d": (4, 1), "2.5d": (8, 2), "3d": (8, 1)}
CLS = {0: "gemm", 1: "gemm-simt", 2: "coll"}


def run(mode, M, h, flags=0):
    p, d = GRIDS[mode]
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)
    bar = threading.Barrier(p)
    out = [None] * p

    def body(r):
        torch.cuda.set_device(0)
        g = api.tp_grid_init(mode, p, r, 0, d, 0, api.TP_TRANSPORT_LOCAL, uid)
        s = torch.cuda.Stream()
        try:
            with torch.cuda.stream(s):
                m = TPMLP(g, M, [(h, h)], flags=flags)
                m.step()  # warm-up
                s.synchronize()
                bar.wait()
                if r == 0:
                    api.tp_prof_reset()
                    api.tp_prof_enable(True)
                bar.wait()
                m.forward()
                s.synchronize()
                bar.wait()
                m.backward()
                s.synchronize()
                bar.wait()
                if r == 0:
                    api.tp_prof_enable(False)
            out[r] = True
        finally:
            s.synchronize()
            api.tp_grid_destroy(g)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    return api.tp_prof_spans()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="3d", choices=sorted(GRIDS))
    ap.add_argument("--M", type=int, default=16384)
    ap.add_argument("--h", type=int, default=16384)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--json")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    spans = run(a.mode, a.M, a.h)
    mine = sorted((s for s in spans if s["rank"] == a.rank), key=lambda s: s["start_ms"])
    t0 = mine[0]["start_ms"] if mine else 0.0
    print(f"{a.mode} M={a.M} h={a.h}: rank {a.rank}, {len(mine)} spans (of {len(spans)})")
    for s in mine:
        v = f"{s['value'] / 1e9:.1f} GFLOP" if s["cls"] < 2 else f"{s['value'] / 1e6:.1f} MB"
        print(f"  {CLS[s['cls']]:9s} {s['start_ms'] - t0:9.3f} -> {s['end_ms'] - t0:9.3f} ms  {v}")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"mode": a.mode, "M": a.M, "h": a.h, "spans": spans}, f)


if __name__ == "__main__":
    main()
