"""Pins of the Cannon forward (oracle/cannon.py): equal to the dense product and to the SUMMA
program on q = 1..4 grids; the skew places X[i,(i+j) mod q] / W[(i+j) mod q, j] (checked by
brute force on iota blocks); the ledger equals the algorithm's count:
skew (q-1) q blocks of X and of W, then (q-1) q^2 blocks of each."""
import numpy as np
import pytest

import synth
from oracle import cannon, dense, programs
from oracle.fabric import Fabric
from oracle.grid import build_grid
from oracle.shards import LayerSpec, gather_full, shard


@pytest.mark.parametrize("q", [1, 2, 3, 4])
def test_cannon_equals_dense_and_summa(q):
    M, K, N = 12 * q, 8 * q, 4 * q
    grid = build_grid("2d", q * q)
    spec = LayerSpec(M, K, N)
    X, W, _, b = synth.layer_inputs(6, M, K, N, with_bias=True)
    fab = Fabric()
    Y = cannon.cannon_fwd(grid, shard(grid, spec, X, "X"), shard(grid, spec, W, "W"),
                          shard(grid, spec, b, "B"), 0.5, fab)
    ref = dense.linear_fwd(X, W, b, alpha=0.5)
    assert np.allclose(gather_full(grid, spec, Y, "Y"), ref, atol=1e-12)
    Ys, _ = programs.layer_fwd(grid, spec, shard(grid, spec, X, "X"), shard(grid, spec, W, "W"),
                               shard(grid, spec, b, "B"), 0.5, Fabric())
    assert np.allclose(gather_full(grid, spec, Y, "Y"), gather_full(grid, spec, Ys, "Y"), atol=1e-12)
    mx, mw = (M // q) * (K // q), (K // q) * (N // q)
    assert fab.ledger.total() == (q - 1) * q * (mx + mw) + (q - 1) * q * q * (mx + mw)


def test_skew_brute_force():
    q = 3
    grid = build_grid("2d", q * q)
    # block (a, c) of X carries the value 10 a + c; of W, 100 a + c
    X = {grid.rank_of((i, j)): np.full((1, 1), 10 * i + j) for i in range(q) for j in range(q)}
    W = {grid.rank_of((i, j)): np.full((1, 1), 100 * i + j) for i in range(q) for j in range(q)}
    fab = Fabric()
    Xh, Wh = dict(X), dict(W)
    for g in grid.groups_along(1):
        Xh.update(cannon._shift(fab, g, Xh, grid.coords(g[0])[0]))
    for g in grid.groups_along(0):
        Wh.update(cannon._shift(fab, g, Wh, grid.coords(g[0])[1]))
    for i in range(q):
        for j in range(q):
            r = grid.rank_of((i, j))
            assert Xh[r][0, 0] == 10 * i + (i + j) % q
            assert Wh[r][0, 0] == 100 * ((i + j) % q) + j


@pytest.mark.parametrize("q", [1, 2, 3, 4])
def test_cannon_bwd_equals_dense_and_summa(q):
    """Cannon's backward (moving accumulators, oracle/cannon.cannon_bwd) == the dense chain rule
    and the SUMMA program, non-square blocks, alpha != 1; the ledger counts the algorithm's
    shifts: W skew (q-1) q blocks + (q-1) q^2 unit shifts, q q^2 accumulator shifts and the
    (q-1) q delivered blocks, likewise for X / dW."""
    M, K, N = 12 * q, 8 * q, 4 * q
    grid = build_grid("2d", q * q)
    spec = LayerSpec(M, K, N)
    X, W, dY, _ = synth.layer_inputs(8, M, K, N)
    fab = Fabric()
    dXs, dWs = cannon.cannon_bwd(grid, shard(grid, spec, dY, "Y"), shard(grid, spec, X, "X"),
                                 shard(grid, spec, W, "W"), 0.5, fab)
    dXr, dWr, _ = dense.linear_bwd(dY, X, W, alpha=0.5)
    assert np.allclose(gather_full(grid, spec, dXs, "X"), dXr, atol=1e-12)
    assert np.allclose(gather_full(grid, spec, dWs, "W"), dWr, atol=1e-12)
    Xs, Ws = shard(grid, spec, X, "X"), shard(grid, spec, W, "W")
    _, sv = programs.layer_fwd(grid, spec, Xs, Ws, None, 0.5, Fabric())
    dXp, dWp, _ = programs.layer_bwd(grid, spec, shard(grid, spec, dY, "Y"), Xs, Ws, 0.5, Fabric(), sv)
    assert np.allclose(gather_full(grid, spec, dXs, "X"), gather_full(grid, spec, dXp, "X"), atol=1e-12)
    assert np.allclose(gather_full(grid, spec, dWs, "W"), gather_full(grid, spec, dWp, "W"), atol=1e-12)
    mb, kq, nq = M // q, K // q, N // q
    mx, mw = mb * kq, kq * nq
    if q == 1:
        assert fab.ledger.total() == 0
    else:
        dx_part = (q - 1) * q * mw + (q - 1) * q * q * mw + q * q * q * mx + (q - 1) * q * mx
        dw_part = (q - 1) * q * mx + (q - 1) * q * q * mx + q * q * q * mw + (q - 1) * q * mw
        assert fab.ledger.total() == dx_part + dw_part


def test_cannon_bwd_one_block_provenance():
    """A single non-zero dY block (i0, j0) must produce dX only in row block i0 and dW only in
    column block j0, each at its owner (the accumulators end where they belong)."""
    q = 3
    grid = build_grid("2d", q * q)
    M, K, N = 6, 9, 12
    spec = LayerSpec(M, K, N)
    X, W, _, _ = synth.layer_inputs(9, M, K, N)
    for i0, j0 in ((0, 2), (2, 1), (1, 0)):
        dY = np.zeros((M, N))
        dY[i0 * 2:(i0 + 1) * 2, j0 * 4:(j0 + 1) * 4] = 1.0
        dXs, dWs = cannon.cannon_bwd(grid, shard(grid, spec, dY, "Y"), shard(grid, spec, X, "X"),
                                     shard(grid, spec, W, "W"))
        dXr, dWr, _ = dense.linear_bwd(dY, X, W)
        assert np.allclose(gather_full(grid, spec, dXs, "X"), dXr, atol=1e-13)
        assert np.allclose(gather_full(grid, spec, dWs, "W"), dWr, atol=1e-13)
