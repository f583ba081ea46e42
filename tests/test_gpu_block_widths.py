"""The Transformer block at the real widths of BASELINE.json's model configs (SURVEY 8(f) NEXT-2
"full ViT-S (C4) and GPT (C5) blocks end to end"; P:L445 ViT, "Jax initialization"):

* configs[3] ViT-S/16: hidden 384, 6 heads of 64, MLP 1536, 197 tokens per image (a ragged
  sequence: 197 is not a multiple of any tile), 8 images (the real batch is 4096: the per-token
  work is the same and a sequence never crosses a shard, so fewer images change no shape but M).
* configs[4] GPT: hidden 8192, 64 heads of 128, MLP 32768, 4 sequences of 512 tokens (the real
  sequence is 2048; 512 keeps the fp64 dense oracle at ~10 TFLOP of CPU work while every
  weight matrix has its real shape).

Each on the grids the north star names (1D, 2D q=2, 2.5D q=2 d=2, 3D l=2, in-process ranks on
cuda:0), bf16, against the dense fp64 oracle block (oracle/block.py, pinned to torch fp64
autograd in tests/test_oracle_block.py), computed once per config. Weights Xavier-uniform, LN
gamma = 1 + U(-0.1, 0.1), beta and biases U(-0.1, 0.1); x and dout U(-1, 1). Bar: relative
Frobenius error <= 1e-2 for the output, dx and every parameter gradient.
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import block as oblock
from oracle.grid import build_grid
from oracle.shards import gather_full

from tp_harness import rel_fro, run_ranks, spec_of, to_np

pytestmark = pytest.mark.gpu

CONFIGS = {"vit_s": dict(h=384, heads=6, F=1536, seq=197, nseq=8),
           "gpt": dict(h=8192, heads=64, F=32768, seq=512, nseq=4)}
GRIDS = [("1d", 1, 1), ("2d", 4, 1), ("2.5d", 8, 2), ("3d", 8, 1)]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def params(seed, h, F):
    bf = lambda t, a, b, s: synth.tensor(seed, t, a, b, scale=s).astype(np.float64)
    xav = lambda a, b: math.sqrt(6.0 / (a + b))
    P = {"W_qkv": bf(0, h, 3 * h, xav(h, 3 * h)), "b_qkv": bf(1, 1, 3 * h, 0.1)[0],
         "W_o": bf(2, h, h, xav(h, h)), "b_o": bf(3, 1, h, 0.1)[0],
         "W_1": bf(4, h, F, xav(h, F)), "b_1": bf(5, 1, F, 0.1)[0],
         "W_2": bf(6, F, h, xav(F, h)), "b_2": bf(7, 1, h, 0.1)[0],
         "be1": bf(9, 1, h, 0.1)[0], "be2": bf(11, 1, h, 0.1)[0]}
    for k, t in (("g1", 8), ("g2", 10)):  # 1 + small, re-quantised to what the GPU stores
        g = 1 + synth.tensor(seed, t, 1, h, scale=0.1).astype(np.float64)[0]
        P[k] = torch.tensor(g).to(torch.bfloat16).double().numpy()
    return P


_REF = {}


def reference(name):
    if name not in _REF:
        c = CONFIGS[name]
        M = c["seq"] * c["nseq"]
        P = params(13, c["h"], c["F"])
        x = synth.tensor(13, 20, M, c["h"]).astype(np.float64)
        dout = synth.tensor(13, 21, M, c["h"]).astype(np.float64)
        out, S = oblock.block_fwd(x, P, c["seq"], c["heads"])
        G = oblock.block_bwd(dout, P, S, c["seq"], c["heads"])
        _REF[name] = (P, x, dout, out, G)
    return _REF[name]


@pytest.mark.parametrize("grid", GRIDS, ids=lambda g: f"{g[0]}-p{g[1]}")
@pytest.mark.parametrize("name", list(CONFIGS))
def test_block_real_widths(api, name, grid):
    from paper_2110_14883_b200.block import TPBlock
    mode, p, d = grid
    c = CONFIGS[name]
    h, F, heads, seq = c["h"], c["F"], c["heads"], c["seq"]
    M = seq * c["nseq"]
    P, x, dout, out_ref, G = reference(name)
    transport = api.TP_TRANSPORT_LOCAL if p > 1 else api.TP_TRANSPORT_NONE
    uid = api.tp_get_unique_id(transport)
    gx = torch.from_numpy(x.astype(np.float32)).cuda().to(torch.bfloat16)
    gd = torch.from_numpy(dout.astype(np.float32)).cuda().to(torch.bfloat16)
    torch.cuda.synchronize()

    def rank_fn(r):
        g = api.tp_grid_init(mode, p, r, 0, d, 0, transport, uid)
        st = torch.cuda.Stream()
        try:
            with torch.cuda.stream(st):
                blk = TPBlock(g, M, h, heads, seq, F=F, dtype="bf16")
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
            del blk
            return res
        finally:
            st.synchronize()
            api.tp_grid_destroy(g)

    per = run_ranks(p, rank_fn, timeout=600)
    torch.cuda.empty_cache()
    gr = build_grid(mode, p, d)
    gat = lambda key, spec, t: gather_full(gr, spec, {r: per[r][key] for r in range(p)}, t)
    sx = spec_of(M, h, 3 * h, 0, 0)
    errs = {"out": rel_fro(gat("out", sx, "X"), out_ref), "dx": rel_fro(gat("dx", sx, "X"), G["x"])}
    specs = {"qkv": spec_of(M, h, 3 * h, 0, 0), "o": spec_of(M, h, h, 1, 1),
             "1": spec_of(M, h, F, 0, 0), "2": spec_of(M, F, h, 1, 1)}
    for k, sp in specs.items():
        errs["dW_" + k] = rel_fro(gat("dW_" + k, sp, "W"), G["W_" + k])
        errs["db_" + k] = rel_fro(np.ravel(gat("db_" + k, sp, "B")), G["b_" + k])
    for k in ("g1", "be1", "g2", "be2"):
        errs["d" + k] = max(rel_fro(per[r]["d" + k],
                                    G[k][per[r]["ln_cols"][0]:per[r]["ln_cols"][0] + per[r]["ln_cols"][1]])
                            for r in range(p))
    print(name, grid, {k: f"{v:.2e}" for k, v in errs.items()})
    bad = {k: v for k, v in errs.items() if v > 1e-2}
    assert not bad, bad
