"""Parity at the BASELINE.json full sizes, in the launch configurations bench.py times.

* configs[1] (C2: two layers, batch 512, hidden 4096): the bench's N=1 program (1D p=1 chain),
  the N=4 program (2D q=2) and the N=8 program (3D l=2), the latter two on 4 / 8 in-process
  ranks of one GPU - every output compared element by element with the dense fp64 oracle.
* configs[2] HEAD (M = h = 16384) and configs[4] (GPT fc1 / fc2 at 16384 tokens): one layer at
  p = 1, tile-stratified samples of Y, dX, dW (one entry per 128x128 output tile) recomputed by
  oracle/sampled.py. The two-layer C3-HEAD chain on the target grids: test_gpu_c3head.py.
* configs[2] literal (batch 64, hidden 16384): 3D l=2 on 8 in-process ranks, full compare.
Inputs are generated on the device by tp_fill (bit-exact with synth, see test_gpu_kernels).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import dense, sampled
from oracle.grid import build_grid
from oracle.shards import LayerSpec, gather_full

from tp_harness import rel_fro, run_ranks, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def chain_inputs(seed, M, layers):
    X = synth.tensor(seed, synth.layer_tid(0, 0), M, layers[0][0]).astype(np.float64)
    Ws = [synth.tensor(seed, synth.layer_tid(i, 1), K, N, scale=synth.xavier_scale(K, N))
          .astype(np.float64) for i, (K, N) in enumerate(layers)]
    dY = synth.tensor(seed, synth.layer_tid(len(layers) - 1, 2), M, layers[-1][1]).astype(np.float64)
    return X, Ws, dY


def oracle_chain(X, Ws, dY):
    acts = [X]
    for W in Ws:
        acts.append(dense.linear_fwd(acts[-1], W))
    dWs = [None] * len(Ws)
    d = dY
    for i in reversed(range(len(Ws))):
        dX, dWs[i], _ = dense.linear_bwd(d, acts[i], Ws[i])
        d = dX
    return acts[-1], d, dWs


def run_chain(api, mode, p, d, M, layers, seed=42, flags=0):
    from paper_2110_14883_b200.mlp import TPMLP
    transport = api.TP_TRANSPORT_LOCAL if p > 1 else api.TP_TRANSPORT_NONE
    uid = api.tp_get_unique_id(transport)

    def rank_fn(r):
        g = api.tp_grid_init(mode, p, r, 0, d, 0, transport, uid)
        s = torch.cuda.Stream()
        try:
            with torch.cuda.stream(s):
                m = TPMLP(g, M, layers, seed=seed, flags=flags)
                m.step()
            s.synchronize()
            return {"Y": to_np(m.Y[-1]), "dX": to_np(m.dX[0]), "dW": [to_np(w) for w in m.dW]}
        finally:
            s.synchronize()
            api.tp_grid_destroy(g)

    return run_ranks(p, rank_fn, timeout=900)


@pytest.mark.parametrize("mode,p,d", [("1d", 1, 1), ("2d", 4, 1), ("3d", 8, 1), ("1d", 8, 1),
                                      ("2.5d", 8, 2)])
def test_c2_two_layer_chain_full(api, mode, p, d):
    M, layers = 512, [(4096, 4096), (4096, 4096)]
    per = run_chain(api, mode, p, d, M, layers)
    X, Ws, dY = chain_inputs(42, M, layers)
    Yr, dXr, dWr = oracle_chain(X, Ws, dY)
    g = build_grid(mode, p, d)
    specs = [LayerSpec(M, K, N, split_1d="row" if i % 2 else "col", parity=i % 2)
             for i, (K, N) in enumerate(layers)]
    Y = gather_full(g, specs[-1], {r: per[r]["Y"] for r in range(p)}, "Y")
    dXg = gather_full(g, specs[0], {r: per[r]["dX"] for r in range(p)}, "X")
    assert rel_fro(Y, Yr) <= 1e-2
    assert rel_fro(dXg, dXr) <= 1e-2
    for i in range(len(layers)):
        dWg = gather_full(g, specs[i], {r: per[r]["dW"][i] for r in range(p)}, "W")
        assert rel_fro(dWg, dWr[i]) <= 1e-2


@pytest.mark.parametrize("name,M,K,N", [("c3head", 16384, 16384, 16384),
                                        ("c5_fc1", 16384, 8192, 32768),
                                        ("c5_fc2", 16384, 32768, 8192)])
def test_single_layer_full_size_sampled(api, name, M, K, N):
    """One layer at p = 1, tile-stratified: one row per 128-row block x one column per
    128-column block of Y, dX and dW (every 128x128 output tile holds a checked entry)."""
    from paper_2110_14883_b200.mlp import TPMLP
    g = api.tp_grid_init("1d", 1, 0)
    r, c, k = (sampled.stratified_indices(s, n) for s, n in ((3, M), (4, N), (5, K)))
    try:
        m = TPMLP(g, M, [(K, N)], seed=7)
        m.step()
        torch.cuda.synchronize()
        rt, ct, kt = (torch.from_numpy(v).cuda() for v in (r, c, k))
        pick = lambda t, a, b: t.index_select(0, a).index_select(1, b).float().cpu().numpy()
        got = {"Y": pick(m.Y[0], rt, ct), "dX": pick(m.dX[0], rt, kt), "dW": pick(m.dW[0], kt, ct)}
    finally:
        api.tp_grid_destroy(g)
    spec = sampled.layer_spec(7, M, K, N)
    ref = {"Y": sampled.y_grid(spec, r, c), "dX": sampled.dx_grid(spec, r, k),
           "dW": sampled.dw_grid(spec, k, c)}
    for key, exp in ref.items():
        err = got[key] - exp
        assert rel_fro(got[key], exp) <= 1e-2, key
        assert np.abs(err).max() <= 5e-2 * np.sqrt(np.mean(exp ** 2)), key


def test_c3_literal_3d_8ranks_full(api):
    """configs[2] literal: batch 64 x hidden 16384, one layer, 3D l=2 (the NVLink-bound corner)."""
    M, layers = 64, [(16384, 16384)]
    per = run_chain(api, "3d", 8, 1, M, layers, seed=11)
    X, Ws, dY = chain_inputs(11, M, layers)
    Yr, dXr, dWr = oracle_chain(X, Ws, dY)
    g = build_grid("3d", 8, 1)
    spec = LayerSpec(M, 16384, 16384, parity=0)
    assert rel_fro(gather_full(g, spec, {r: per[r]["Y"] for r in range(8)}, "Y"), Yr) <= 1e-2
    assert rel_fro(gather_full(g, spec, {r: per[r]["dX"] for r in range(8)}, "X"), dXr) <= 1e-2
    assert rel_fro(gather_full(g, spec, {r: per[r]["dW"][0] for r in range(8)}, "W"), dWr[0]) <= 1e-2


@pytest.mark.parametrize("variant", ["fused-2d", "depth-sharded-2.5d", "fused-depth-sharded-2.5d",
                                     "solomonik-2.5d"])
def test_c2_chain_full_variants(api, variant):
    """configs[1] at full size through the variant schedules: the fused peer-panel 2D (q=2 on 4
    ranks), the 2.5D with depth-sharded weights (collective and fused requested; C2's 128-row
    plane blocks take the collective path), and Solomonik's 2.5D (q=2, d=2 on 8 ranks)."""
    from oracle import solomonik as so
    M, layers = 512, [(4096, 4096), (4096, 4096)]
    mode, p, d, flags = {"fused-2d": ("2d", 4, 1, api.TP_FLAG_PEER_FUSED),
                         "depth-sharded-2.5d": ("2.5d", 8, 2, api.TP_FLAG_W25_DEPTH_SHARDED),
                         "fused-depth-sharded-2.5d": ("2.5d", 8, 2, api.TP_FLAG_W25_DEPTH_SHARDED
                                                      | api.TP_FLAG_PEER_FUSED),
                         "solomonik-2.5d": ("2.5d", 8, 2, api.TP_FLAG_SOLOMONIK)}[variant]
    per = run_chain(api, mode, p, d, M, layers, flags=flags)
    X, Ws, dY = chain_inputs(42, M, layers)
    Yr, dXr, dWr = oracle_chain(X, Ws, dY)
    g = build_grid(mode, p, d)
    sharded = bool(flags & api.TP_FLAG_W25_DEPTH_SHARDED)
    specs = [LayerSpec(M, K, N, w_depth_sharded=sharded) for K, N in layers]
    gf = (lambda sp, sh, t: so.gather_full(g, sp, sh, t)) if flags & api.TP_FLAG_SOLOMONIK else \
        (lambda sp, sh, t: gather_full(g, sp, sh, t))
    assert rel_fro(gf(specs[-1], {r: per[r]["Y"] for r in range(p)}, "Y"), Yr) <= 1e-2
    assert rel_fro(gf(specs[0], {r: per[r]["dX"] for r in range(p)}, "X"), dXr) <= 1e-2
    for i in range(len(layers)):
        assert rel_fro(gf(specs[i], {r: per[r]["dW"][i] for r in range(p)}, "W"), dWr[i]) <= 1e-2
