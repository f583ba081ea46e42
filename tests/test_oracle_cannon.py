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
