"""Fused peer-panel schedule vs the collective schedule, all ranks on ONE GPU (LOCAL transport,
one host thread per rank). Not a multi-GPU number: every rank shares the same SMs and HBM, so
this measures the work each schedule puts on the device (copies, partial passes, launches) —
the fused path drops the panel broadcasts / gathers / reduce-scatters entirely.

    python tools/fused_bench.py [--mode 2d|3d|2.5d] [--M 4096] [--hidden 4096] [--steps 10]
Prints one JSON line per schedule: device ms per step (max over ranks, CUDA events on each
rank's stream between two host barriers).
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

GRIDS = {"1d": (4, 1), "2d": (4, 1), "2.5d": (8, 2), "3d": (8, 1)}


def run(mode, M, h, steps, warmup, flags):
    p, d = GRIDS[mode]
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)
    bar = threading.Barrier(p)
    out = [None] * p
    err = [None] * p

    def body(r):
        try:
            torch.cuda.set_device(0)
            g = api.tp_grid_init(mode, p, r, 0, d, 0, api.TP_TRANSPORT_LOCAL, uid)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                m = TPMLP(g, M, [(h, h), (h, h)], flags=flags)
                for _ in range(warmup):
                    m.step()
                s.synchronize()
                bar.wait()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                for _ in range(steps):
                    m.step()
                e1.record(s)
                s.synchronize()
                out[r] = e0.elapsed_time(e1) / steps
                bar.wait()
            api.tp_grid_destroy(g)
        except BaseException as e:  # noqa: BLE001
            err[r] = e
            bar.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in err:
        if e is not None:
            raise e
    return max(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="2d", choices=sorted(GRIDS))
    ap.add_argument("--M", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    flops = 2 * 6.0 * a.M * a.hidden * a.hidden
    for name, flags in (("collective", 0), ("fused", api.TP_FLAG_PEER_FUSED)):
        ms = run(a.mode, a.M, a.hidden, a.steps, a.warmup, flags)
        print(json.dumps({"mode": a.mode, "schedule": name, "M": a.M, "hidden": a.hidden,
                          "ms_per_step": round(ms, 4),
                          "tflops_one_gpu": round(flops / ms / 1e9, 1)}), flush=True)


if __name__ == "__main__":
    main()
