"""Test harness: run a multi-rank grid on ONE GPU through the C ABI's in-process
transport (one host thread per rank, all ranks on cuda:0), and compare against the oracle.

Inputs come from `synth` (the shared seeded generator); expected values only from `oracle/`.
"""
from __future__ import annotations

import threading

import numpy as np
import torch

import synth
from oracle import dense, programs
from oracle.fabric import Fabric
from oracle.grid import build_grid
from oracle.shards import LayerSpec, gather_full, shard as oshard

TORCH_DT = {"bf16": torch.bfloat16, "fp32": torch.float32}


def run_ranks(p, fn, timeout=300):
    """fn(rank) in p threads; returns [result...]; re-raises the first exception."""
    out, errs = [None] * p, [None] * p

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs[r] = e

    ts = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(p)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
        if t.is_alive():
            raise TimeoutError("rank thread hung (collective mismatch?)")
    for e in errs:
        if e is not None:
            raise e
    return out


def to_dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to("cuda").to(TORCH_DT[dtype])


def to_np(t):
    return t.float().cpu().numpy().astype(np.float64)


def spec_of(M, K, N, split_1d=0, parity=0, flags=0):
    return LayerSpec(M, K, N, split_1d="row" if split_1d else "col", parity=parity,
                     w_depth_sharded=bool(flags & 1))


def tp_layer(api, mode, p, d, M, K, N, X, W, dY, b=None, dtype="bf16", split_1d=0, parity=0,
             flags=0, alpha=1.0, want_dx=True):
    """Run fwd+bwd of one layer on p in-process ranks. Global inputs are numpy fp32 (already
    quantised). Returns per-rank dicts of numpy shards."""
    transport = api.TP_TRANSPORT_LOCAL if p > 1 else api.TP_TRANSPORT_NONE
    uid = api.tp_get_unique_id(transport)
    gX, gW, gdY = to_dev(X, dtype), to_dev(W, dtype), to_dev(dY, dtype)
    gb = to_dev(b[None, :], dtype)[0].contiguous() if b is not None else None
    torch.cuda.synchronize()
    bar = threading.Barrier(p)

    def rank_fn(r):
        g = api.tp_grid_init(mode, p, r, 0, d, 0, transport, uid)
        s = torch.cuda.Stream()
        try:
            with torch.cuda.stream(s):
                ds = api.desc(M, K, N, dtype, split_1d, parity, flags, alpha)
                ext = {t: api.tp_shard_extent(g, ds, t) for t in ("X", "W", "Y", "B")}
                mk = lambda t: torch.empty(ext[t][1], ext[t][3], device="cuda", dtype=TORCH_DT[dtype])
                x, w, y, dy = mk("X"), mk("W"), mk("Y"), mk("Y")
                dx = torch.empty_like(x) if want_dx else None
                wsb, svb = api.tp_workspace_size(g, ds)
                ws = torch.empty(max(wsb, 1), device="cuda", dtype=torch.uint8)
                if flags & api.TP_FLAG_PEER_FUSED:  # peers read / write these directly
                    for t in (x, w, dy, y, dx, ws):
                        if t is not None:
                            api.tp_register_buffer(g, t)
                api.tp_pack(g, ds, "X", gX, x)
                api.tp_pack(g, ds, "W", gW, w)
                api.tp_pack(g, ds, "Y", gdY, dy)
                bias = None
                if gb is not None:
                    bias = torch.empty(ext["B"][3], device="cuda", dtype=TORCH_DT[dtype])
                    api.tp_pack(g, ds, "B", gb, bias)
                sv = torch.empty(svb, device="cuda", dtype=torch.uint8) if svb else None
                s.synchronize()
                bar.wait(120)  # count the launches of all ranks' forward calls (rank 0 reads)
                n0 = api.tp_launch_count()
                bar.wait(120)
                st0 = api.tp_peer_staged_bytes(g)
                api.tp_linear_fwd(g, ds, x, w, bias, y, sv, ws)
                staged_fwd = api.tp_peer_staged_bytes(g) - st0
                bar.wait(120)
                n_fwd = api.tp_launch_count() - n0
                bar.wait(120)  # no rank enqueues its backward before every rank has read the count
                dw = torch.empty_like(w)
                db = torch.empty(ext["B"][3], device="cuda", dtype=TORCH_DT[dtype])
                api.tp_linear_bwd(g, ds, dy, x, w, sv, dx, dw, db, ws)
            s.synchronize()
            res = {"Y": to_np(y), "dW": to_np(dw), "dB": to_np(db), "n_fwd": n_fwd,
                   "staged_fwd": staged_fwd, "staged_bwd": api.tp_peer_staged_bytes(g) - st0 - staged_fwd}
            if want_dx:
                res["dX"] = to_np(dx)
            return res
        finally:
            s.synchronize()
            api.tp_grid_destroy(g)

    return run_ranks(p, rank_fn)


def gather(mode, p, d, spec, per_rank, key, tensor):
    g = build_grid(mode, p, d)
    return gather_full(g, spec, {r: per_rank[r][key] for r in range(p)}, tensor)


def oracle_layer(mode, p, d, spec, X, W, dY, b=None, alpha=1.0):
    """Expected global (Y, dX, dW, db) from the oracle's rank-by-rank program (fp64)."""
    g = build_grid(mode, p, d)
    fab = Fabric()
    Xs, Ws = oshard(g, spec, X, "X"), oshard(g, spec, W, "W")
    bs = oshard(g, spec, b, "B") if b is not None else None
    Ys, sv = programs.layer_fwd(g, spec, Xs, Ws, bs, alpha, fab)
    dXs, dWs, dbs = programs.layer_bwd(g, spec, oshard(g, spec, dY, "Y"), Xs, Ws, alpha, fab, sv)
    return (gather_full(g, spec, Ys, "Y"), gather_full(g, spec, dXs, "X"),
            gather_full(g, spec, dWs, "W"), gather_full(g, spec, dbs, "B"))


def rel_fro(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    n = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (n if n > 0 else 1.0))


def chain_reference(seed, M, layers):
    """Dense fp64 (Y_last, dX, dW_0, dW_1, ...) of a TPMLP chain with the synth recipe of
    paper_2110_14883_b200/mlp.py (X of layer 0, Xavier W_i, dY of the last layer)."""
    X = synth.tensor(seed, synth.layer_tid(0, synth.TID_X), M, layers[0][0]).astype(np.float64)
    Ws = [synth.tensor(seed, synth.layer_tid(i, synth.TID_W), K, N, scale=synth.xavier_scale(K, N))
          .astype(np.float64) for i, (K, N) in enumerate(layers)]
    dY = synth.tensor(seed, synth.layer_tid(len(layers) - 1, synth.TID_DY), M,
                      layers[-1][1]).astype(np.float64)
    acts = [X]
    for W in Ws:
        acts.append(dense.linear_fwd(acts[-1], W))
    d, dWs = dY, [None] * len(Ws)
    for i in reversed(range(len(Ws))):
        d, dWs[i], _ = dense.linear_bwd(d, acts[i], Ws[i])
    return (acts[-1], d, *dWs)
