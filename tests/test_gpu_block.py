"""A whole pre-LN Transformer block (LN, QKV, attention core, projection, residual, LN, fc1 +
GeLU, fc2, residual) forward + backward on every TP mode against the oracle block
(oracle/block.py, pinned to torch fp64 autograd in tests/test_oracle_block.py). SURVEY 8(f)
NEXT-2. In-process ranks on cuda:0."""
import numpy as np
import pytest
import torch

import synth
from oracle import block as oblock
from oracle.grid import build_grid
from oracle.shards import gather_full

from tp_harness import rel_fro, run_ranks, spec_of, to_np

pytestmark = pytest.mark.gpu

GRIDS = [("1d", 1, 1, 0), ("1d", 2, 1, 0), ("2d", 4, 1, 0), ("2.5d", 4, 1, 0), ("2.5d", 8, 2, 0),
         ("2.5d", 8, 2, 1), ("3d", 8, 1, 0)]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def params(seed, h, F, dtype):
    q = "bf16" if dtype == "bf16" else "fp32"
    r = lambda t, a, b, s: synth.tensor(seed, t, a, b, dtype=q).astype(np.float64) * s
    P = {"W_qkv": r(0, h, 3 * h, 0.1), "b_qkv": r(1, 1, 3 * h, 0.1)[0], "W_o": r(2, h, h, 0.1),
         "b_o": r(3, 1, h, 0.1)[0], "W_1": r(4, h, F, 0.1), "b_1": r(5, 1, F, 0.1)[0],
         "W_2": r(6, F, h, 0.1), "b_2": r(7, 1, h, 0.1)[0], "g1": 1 + r(8, 1, h, 0.1)[0],
         "be1": r(9, 1, h, 0.1)[0], "g2": 1 + r(10, 1, h, 0.1)[0], "be2": r(11, 1, h, 0.1)[0]}
    if dtype == "bf16":  # gamma = 1 + small is re-quantised to what the GPU stores
        for k in ("g1", "g2"):
            P[k] = torch.tensor(P[k]).to(torch.bfloat16).double().numpy()
    return P


@pytest.mark.parametrize("grid", GRIDS, ids=lambda g: f"{g[0]}-p{g[1]}" + ("-wsharded" if g[3] else ""))
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_block_vs_oracle(api, grid, dtype):
    from paper_2110_14883_b200.block import TPBlock
    mode, p, d, wflags = grid
    seq, heads, dh, B = 64, 4, 32, 8
    h, F, M = heads * dh, 256, B * seq
    P = params(7, h, F, dtype)
    q = "bf16" if dtype == "bf16" else "fp32"
    x = synth.tensor(7, 20, M, h, dtype=q).astype(np.float64)
    dout = synth.tensor(7, 21, M, h, dtype=q).astype(np.float64)
    transport = api.TP_TRANSPORT_LOCAL if p > 1 else api.TP_TRANSPORT_NONE
    uid = api.tp_get_unique_id(transport)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    gx = torch.from_numpy(x.astype(np.float32)).cuda().to(tdt)
    gd = torch.from_numpy(dout.astype(np.float32)).cuda().to(tdt)
    torch.cuda.synchronize()

    def rank_fn(r):
        g = api.tp_grid_init(mode, p, r, 0, d, 0, transport, uid)
        st = torch.cuda.Stream()
        try:
            with torch.cuda.stream(st):
                blk = TPBlock(g, M, h, heads, seq, F=F, dtype=dtype, flags=wflags)
                blk.load(P)
                api.tp_pack(g, blk.dq, "X", gx, blk.x)
                api.tp_pack(g, blk.dq, "X", gd, blk.dout)
                blk.step()
            st.synchronize()
            res = {"out": to_np(blk.out), "dx": to_np(blk.dx), "ln_cols": blk.ln_cols}
            for k in blk.dW:
                res["dW_" + k] = to_np(blk.dW[k])
                res["db_" + k] = to_np(blk.db[k])
            for k in blk.dln:
                res["d" + k] = to_np(blk.dln[k])
            return res
        finally:
            st.synchronize()
            api.tp_grid_destroy(g)

    per = run_ranks(p, rank_fn)
    out_ref, S = oblock.block_fwd(x, P, seq, heads)
    G = oblock.block_bwd(dout, P, S, seq, heads)
    gr = build_grid(mode, p, d)
    sx = spec_of(M, h, 3 * h, 0, 0, wflags)
    tol = 1e-5 if dtype == "fp32" else 1e-2          # the north star's bars
    gat = lambda key, spec, t: gather_full(gr, spec, {r: per[r][key] for r in range(p)}, t)
    errs = {"out": rel_fro(gat("out", sx, "X"), out_ref), "dx": rel_fro(gat("dx", sx, "X"), G["x"])}
    specs = {"qkv": spec_of(M, h, 3 * h, 0, 0, wflags), "o": spec_of(M, h, h, 1, 1, wflags),
             "1": spec_of(M, h, F, 0, 0, wflags), "2": spec_of(M, F, h, 1, 1, wflags)}
    for k, sp in specs.items():
        errs["dW_" + k] = rel_fro(gat("dW_" + k, sp, "W"), G["W_" + k])
        errs["db_" + k] = rel_fro(np.ravel(gat("db_" + k, sp, "B")), G["b_" + k])
    for k in ("g1", "be1", "g2", "be2"):
        errs["d" + k] = max(rel_fro(per[r]["d" + k], G[k][per[r]["ln_cols"][0]:
                                                           per[r]["ln_cols"][0] + per[r]["ln_cols"][1]])
                            for r in range(p))
    print(dtype, grid, {k: f"{v:.2e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if v > tol}
    assert not bad, bad
