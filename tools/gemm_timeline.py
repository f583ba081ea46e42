"""Per-unit timeline of the CTA-pair GEMM (diagnostics build: TP_NVCC_FLAGS=-DTP_TIMELINE=1).

    TP_NVCC_FLAGS=-DTP_TIMELINE=1 python tools/gemm_timeline.py 4096x4096x512 TN [--hot] [--group]

For every leader CTA: when each unit's first MMA was issued, when its accumulator commit was
issued, when the epilogue (warp 2) saw it and when it released TMEM, in SM cycles from the CTA's
entry; plus warp 2's epilogue phase sums (TMEM load, staging-buffer wait, stage + fence, store
issue). --group runs the C2 backward pair (dX = dY W^T, dW = X^T dY) as one grouped launch.
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
    shp = sys.argv[1] if len(sys.argv) > 1 else "4096x4096x512"
    op = sys.argv[2] if len(sys.argv) > 2 else "TN"
    hot = "--hot" in sys.argv
    group = "--group" in sys.argv
    M, N, K = map(int, shp.split("x"))
    ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    flush = torch.empty(256 << 20, device="cuda", dtype=torch.uint8)
    tr = torch.zeros(300 * 16 + 300 * 128, device="cuda", dtype=torch.int64)
    if group:  # one C2-style layer's backward (dX and dW as one grouped launch): rows M, K x N
        from paper_2110_14883_b200.mlp import TPMLP
        g = api.tp_grid_init("1d", 1, 0, 0, 1, 0, api.TP_TRANSPORT_NONE)
        mlp = TPMLP(g, M, [(K, N)])
        mlp.forward()
        run = mlp.backward
    else:
        ta, tb = OPS[op]
        A = torch.randn(*((K, M) if ta else (M, K)), device="cuda").to(torch.bfloat16)
        B = torch.randn(*((N, K) if tb else (K, N)), device="cuda").to(torch.bfloat16)
        D = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        run = lambda: api.tp_gemm(ta, tb, M, N, K, "bf16", A, A.shape[1], B, B.shape[1], None, N, D,
                                  N, "bf16", ws=ws)
    run()
    torch.cuda.synchronize()
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
    base = tr[: 300 * 16].view(-1, 16).cpu()
    tl = tr[300 * 16:].view(-1, 128).cpu()
    live = tl[:, 0] > 0
    ctas = int(live.sum())
    out = {"shape": shp, "op": op, "group": group, "hot": hot, "ctas": ctas,
           "diag": os.environ.get("TP_GEMM_EPI_DIAG", "0"),
           "event_us": round(e0.elapsed_time(e1) * 1000, 2)}
    ent, pro, ext = base[:, 7].double(), base[:, 8].double(), base[:, 9].double()
    lv = base[:, 1] > 0
    if not bool(lv.any()):
        print(json.dumps({"shape": shp, "op": op, "error": "no pair-kernel CTAs traced (1-CTA kernel?)"}))
        return
    out["span_us"] = round(float(ext[lv].max() - ent[lv].min()) / 1000, 2)
    out["sm_mhz"] = round(float(((base[lv, 11] - base[lv, 10]).double() / (ext[lv] - ent[lv])).mean()) * 1000, 0)
    rows = []
    for c in range(tl.shape[0]):
        r = tl[c]
        if r[0] <= 0 or r[8] <= 0:  # leaders only (they issue the MMAs)
            continue
        e = int(r[0])
        units = []
        for i in range(16):
            if r[8 + i] <= 0:
                break
            units.append([int(r[8 + i]) - e, int(r[24 + i]) - e,
                          int(r[40 + i]) - e if r[40 + i] > 0 else -1,
                          int(r[56 + i]) - e if r[56 + i] > 0 else -1])
        rows.append({"cta": c, "prologue": int(r[1]) - e, "exit": int(r[2]) - e,
                     "tma_first": int(r[3]) - e, "tma_last": int(r[4]) - e, "units": units,
                     "epi_tmem": int(r[72]), "epi_wait_buf": int(r[73]), "epi_stage": int(r[74]),
                     "epi_store": int(r[75]), "epi_setup": int(r[76]), "epi_finish": int(r[77]),
                     "epi_release": int(r[78])})
    rows.sort(key=lambda x: -x["exit"])
    out["slowest"] = rows[:3]
    out["median"] = rows[len(rows) // 2] if rows else None
    n = max(len(rows), 1)
    for k in ("prologue", "exit", "tma_first", "epi_tmem", "epi_wait_buf", "epi_stage", "epi_store",
              "epi_setup", "epi_finish", "epi_release"):
        out["mean_" + k] = round(sum(x[k] for x in rows) / n)
    # mean epilogue duration per unit (saw -> released) and MMA span per unit (first MMA -> commit)
    epi = [u[3] - u[2] for x in rows for u in x["units"] if u[2] >= 0 and u[3] >= 0]
    mma = [u[1] - u[0] for x in rows for u in x["units"]]
    lag = [u[2] - u[1] for x in rows for u in x["units"] if u[2] >= 0]
    out["mean_unit_epi"] = round(sum(epi) / max(len(epi), 1))
    out["mean_unit_mma_issue"] = round(sum(mma) / max(len(mma), 1))
    out["mean_commit_to_epi"] = round(sum(lag) / max(len(lag), 1))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
