"""Pins of the LayerNorm oracle (oracle/layernorm.py) to things other than itself: a
pure-Python loop, PyTorch's fp64 layer_norm (library routine) and its autograd, central
finite differences, the normalisation invariants, and the rank-by-rank programs equal to the
dense definition on every layout."""
import numpy as np
import pytest
import torch

import synth
from oracle import layernorm as ln
from oracle.fabric import Fabric
from oracle.grid import build_grid
from oracle.shards import LayerSpec, gather_full, shard


def _inputs(seed, M, H):
    X = synth.tensor(seed, 0, M, H, dtype="fp32").astype(np.float64) * 3 + 0.5
    g = 1 + 0.25 * synth.tensor(seed, 1, 1, H, dtype="fp32")[0].astype(np.float64)
    b = 0.1 * synth.tensor(seed, 2, 1, H, dtype="fp32")[0].astype(np.float64)
    dY = synth.tensor(seed, 3, M, H, dtype="fp32").astype(np.float64)
    return X, g, b, dY


def test_fwd_matches_python_loops():
    X, g, b, _ = _inputs(1, 5, 7)
    eps = 1e-5
    Y, mu, rstd = ln.ln_fwd(X, g, b, eps)
    for r in range(5):
        m = sum(X[r]) / 7
        v = sum((x - m) ** 2 for x in X[r]) / 7
        for c in range(7):
            ref = (X[r][c] - m) / (v + eps) ** 0.5 * g[c] + b[c]
            assert abs(Y[r][c] - ref) < 1e-12


def test_matches_torch_fp64_and_autograd():
    X, g, b, dY = _inputs(2, 12, 40)
    eps = 1e-5
    Y, mu, rstd = ln.ln_fwd(X, g, b, eps)
    tX = torch.tensor(X, requires_grad=True)
    tg = torch.tensor(g, requires_grad=True)
    tb = torch.tensor(b, requires_grad=True)
    tY = torch.nn.functional.layer_norm(tX, (40,), tg, tb, eps)
    assert np.allclose(Y, tY.detach().numpy(), rtol=0, atol=1e-12)
    tY.backward(torch.tensor(dY))
    dX, dg, db = ln.ln_bwd(dY, X, g, mu, rstd)
    assert np.allclose(dX, tX.grad.numpy(), rtol=0, atol=1e-12)
    assert np.allclose(dg, tg.grad.numpy(), rtol=0, atol=1e-12)
    assert np.allclose(db, tb.grad.numpy(), rtol=0, atol=1e-12)


def test_finite_differences():
    X, g, b, dY = _inputs(3, 4, 9)
    eps = 1e-3
    Y, mu, rstd = ln.ln_fwd(X, g, b, eps)
    dX, dg, db = ln.ln_bwd(dY, X, g, mu, rstd)
    loss = lambda X_, g_, b_: float((ln.ln_fwd(X_, g_, b_, eps)[0] * dY).sum())
    h = 1e-6
    for (r, c) in [(0, 0), (1, 4), (3, 8)]:
        E = np.zeros_like(X)
        E[r, c] = h
        fd = (loss(X + E, g, b) - loss(X - E, g, b)) / (2 * h)
        assert abs(fd - dX[r, c]) < 1e-6
    for c in [0, 5]:
        e = np.zeros_like(g)
        e[c] = h
        assert abs((loss(X, g + e, b) - loss(X, g - e, b)) / (2 * h) - dg[c]) < 1e-6
        assert abs((loss(X, g, b + e) - loss(X, g, b - e)) / (2 * h) - db[c]) < 1e-6


def test_invariants():
    X, g, b, _ = _inputs(4, 6, 32)
    Y, mu, rstd = ln.ln_fwd(X, np.ones(32), np.zeros(32), 0.0)
    assert np.allclose(Y.mean(axis=1), 0, atol=1e-12)          # centred rows
    assert np.allclose((Y ** 2).mean(axis=1), 1, atol=1e-12)   # unit variance at eps = 0
    Y2, _, _ = ln.ln_fwd(3.5 * X - 7.0, g, b, 0.0)             # row affine invariance
    assert np.allclose(Y2, ln.ln_fwd(X, g, b, 0.0)[0], atol=1e-10)
    C = np.tile(np.arange(32.0), (3, 1)) * 0 + 2.0             # constant rows -> beta
    assert np.allclose(ln.ln_fwd(C, g, b, 1e-5)[0], b[None, :], atol=1e-12)


LAYOUTS = [("1d", 1, 1, "col", 0, "X"), ("1d", 4, 1, "col", 0, "Y"), ("1d", 4, 1, "row", 0, "X"),
           ("1d", 4, 1, "row", 0, "Y"), ("2d", 4, 1, "col", 0, "X"), ("2d", 9, 1, "col", 0, "Y"),
           ("2.5d", 8, 2, "col", 0, "X"), ("2.5d", 8, 2, "col", 0, "Y"),
           ("3d", 8, 1, "col", 0, "X"), ("3d", 8, 1, "col", 1, "X"),
           ("3d", 8, 1, "col", 0, "Y"), ("3d", 8, 1, "col", 1, "Y")]


@pytest.mark.parametrize("lay", LAYOUTS, ids=lambda l: "-".join(map(str, l)))
def test_rank_programs_equal_dense(lay):
    mode, p, d, split, par, tensor = lay
    M, K, N = 72, 36, 72
    grid = build_grid(mode, p, d)
    spec = LayerSpec(M, K, N, split_1d=split, parity=par)
    H = K if tensor == "X" else N
    X, g, b, dY = _inputs(5, M, H)
    eps = 1e-5
    Yd, mu, rstd = ln.ln_fwd(X, g, b, eps)
    dXd, dgd, dbd = ln.ln_bwd(dY, X, g, mu, rstd)
    fab = Fabric()
    Xs = shard(grid, spec, X, tensor)
    ex = ln.groups(grid, spec, tensor)[0]
    gs = {r: g[e.col0:e.col0 + e.cols] for r, e in ex.items()}   # gamma / beta: column blocks
    bs = {r: b[e.col0:e.col0 + e.cols] for r, e in ex.items()}
    Ys, saved = ln.ln_fwd_ranks(grid, spec, tensor, Xs, gs, bs, eps, fab)
    assert np.allclose(gather_full(grid, spec, Ys, tensor), Yd, atol=1e-12)
    dYs = shard(grid, spec, dY, tensor)
    dXs, dg, db = ln.ln_bwd_ranks(grid, spec, tensor, dYs, Xs, gs, saved, fab)
    assert np.allclose(gather_full(grid, spec, dXs, tensor), dXd, atol=1e-12)
    for r in range(p):
        e = ex[r]
        assert np.allclose(dg[r], dgd[e.col0:e.col0 + e.cols], atol=1e-11)
        assert np.allclose(db[r], dbd[e.col0:e.col0 + e.cols], atol=1e-11)


def test_row_stat_volume_is_two_reductions_per_row_block():
    """Forward all-reduces 2 row vectors per row group (sum, centred squares): with the ring
    ledger each group of g members moves 2 * 2(g-1) * rows elements."""
    grid = build_grid("2d", 4)
    spec = LayerSpec(8, 8, 8)
    X, g, b, _ = _inputs(6, 8, 8)
    fab = Fabric()
    ex = ln.groups(grid, spec, "X")[0]
    ln.ln_fwd_ranks(grid, spec, "X", shard(grid, spec, X, "X"),
                    {r: g[e.col0:e.col0 + e.cols] for r, e in ex.items()},
                    {r: b[e.col0:e.col0 + e.cols] for r, e in ex.items()}, 1e-5, fab)
    # 2 row groups x 2 reductions x ring 2(g-1) m with g = 2, m = 4 rows
    assert fab.ledger.total() == 2 * 2 * 2 * 1 * 4
