"""LayerNorm over the hidden (column) dimension of a tensor-parallel activation shard.
TEST INFRASTRUCTURE ONLY (imported by tests/ only).

SURVEY 8(f) NEXT-2: "LayerNorm (row statistics across the column axis)" -- the layer the
paper's parallelized Transformer places around every linear ("parallelized model
components", P:L445 ViT blocks). The paper gives no formula; this is the textbook definition
(Ba et al. 2016), per row r of X [M, H]:

    mu_r   = (1/H) sum_c X[r,c]
    var_r  = (1/H) sum_c (X[r,c] - mu_r)^2            (biased, as in every framework)
    xhat   = (X[r,c] - mu_r) / sqrt(var_r + eps)
    Y      = xhat * gamma[c] + beta[c]

    backward, g = dY * gamma:
    dX     = rstd_r * (g - mean_c(g) - xhat * mean_c(g * xhat))
    dgamma = sum_r dY * xhat,   dbeta = sum_r dY

Rank-by-rank program (`ln_fwd_ranks` / `ln_bwd_ranks`): a rank holds a block
(row0, rows, col0, cols) of X in the layout `tensor` of a layer (shards.extent). Row
statistics need the sums over ALL columns of its rows: they are all-reduced over the distinct
column blocks of those rows (two passes: sum -> mean, then centred squares -> variance,
reading N1 in DESIGN.md). dgamma / dbeta of a column block are all-reduced over the distinct
row blocks holding those columns. Replicated blocks count once. The groups are derived here
from the shard extents alone (equal (row0, rows) / equal (col0, cols)), independently of any
grid axis logic.
"""
from __future__ import annotations

import numpy as np

from .fabric import Fabric
from .grid import Grid
from .shards import LayerSpec, extent


def ln_fwd(X, gamma, beta, eps):
    X = np.asarray(X, np.float64)
    mu = X.mean(axis=1)
    var = ((X - mu[:, None]) ** 2).mean(axis=1)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (X - mu[:, None]) * rstd[:, None]
    return xhat * np.asarray(gamma, np.float64)[None, :] + np.asarray(beta, np.float64)[None, :], mu, rstd


def ln_bwd(dY, X, gamma, mu, rstd):
    dY = np.asarray(dY, np.float64)
    X = np.asarray(X, np.float64)
    xhat = (X - mu[:, None]) * rstd[:, None]
    g = dY * np.asarray(gamma, np.float64)[None, :]
    dX = rstd[:, None] * (g - g.mean(axis=1, keepdims=True) - xhat * (g * xhat).mean(axis=1, keepdims=True))
    return dX, (dY * xhat).sum(axis=0), dY.sum(axis=0)


def groups(grid: Grid, spec: LayerSpec, tensor: str):
    """rank -> (row group, column group). Row group: the ranks holding the same rows
    (replicas included); column group: the ranks holding the same columns. A reduction over
    a group counts each distinct block once (`reps`)."""
    ex = {r: extent(grid, spec, r, tensor) for r in range(grid.world)}
    row_g, col_g = {}, {}
    for r, e in ex.items():
        row_g[r] = [s for s in range(grid.world) if (ex[s].row0, ex[s].rows) == (e.row0, e.rows)]
        col_g[r] = [s for s in range(grid.world) if (ex[s].col0, ex[s].cols) == (e.col0, e.cols)]
    return ex, row_g, col_g


def reps(ex, members, key):
    """The lowest rank of each distinct block (by `key` of the extent) among `members`."""
    out = {}
    for s in members:
        out.setdefault(key(ex[s]), s)
    return sorted(out.values())


def _allreduce_distinct(fab, ex, members, key, parts):
    """Sum of `parts` over the distinct blocks among `members` (one ring all-reduce over a
    representative per block); every member receives the sum."""
    rs = reps(ex, members, key)
    total = fab.all_reduce(rs, {s: parts[s] for s in rs})[rs[0]] if len(rs) > 1 else parts[rs[0]]
    return {s: np.array(total, copy=True) for s in members}


def ln_fwd_ranks(grid: Grid, spec: LayerSpec, tensor: str, Xs: dict, gammas: dict, betas: dict,
                 eps: float, fab: Fabric):
    """Per-rank Y shards and saved (mu, rstd) of the local rows."""
    ex, row_g, _ = groups(grid, spec, tensor)
    H = spec.K if tensor == "X" else spec.N
    ckey = lambda e: (e.col0, e.cols)
    # pass 1: partial row sums over the local columns, summed over the column blocks
    part = {r: np.asarray(Xs[r], np.float64).sum(axis=1) for r in range(grid.world)}
    mu = {}
    for r in range(grid.world):
        if r not in mu:
            for s, v in _allreduce_distinct(fab, ex, row_g[r], ckey, part).items():
                mu[s] = v / H
    # pass 2: partial centred sums of squares
    part2 = {r: ((np.asarray(Xs[r], np.float64) - mu[r][:, None]) ** 2).sum(axis=1)
             for r in range(grid.world)}
    var = {}
    for r in range(grid.world):
        if r not in var:
            for s, v in _allreduce_distinct(fab, ex, row_g[r], ckey, part2).items():
                var[s] = v / H
    Ys, saved = {}, {}
    for r in range(grid.world):
        rstd = 1.0 / np.sqrt(var[r] + eps)
        xhat = (np.asarray(Xs[r], np.float64) - mu[r][:, None]) * rstd[:, None]
        Ys[r] = xhat * np.asarray(gammas[r], np.float64)[None, :] + np.asarray(betas[r], np.float64)[None, :]
        saved[r] = (mu[r], rstd)
    return Ys, saved


def ln_bwd_ranks(grid: Grid, spec: LayerSpec, tensor: str, dYs: dict, Xs: dict, gammas: dict,
                 saved: dict, fab: Fabric):
    """Per-rank dX shards and the column-block dgamma / dbeta (all-reduced over the ranks
    holding the same columns and different rows)."""
    ex, row_g, col_g = groups(grid, spec, tensor)
    H = spec.K if tensor == "X" else spec.N
    xh, gg, pa, pb = {}, {}, {}, {}
    for r in range(grid.world):
        mu, rstd = saved[r]
        xh[r] = (np.asarray(Xs[r], np.float64) - mu[:, None]) * rstd[:, None]
        gg[r] = np.asarray(dYs[r], np.float64) * np.asarray(gammas[r], np.float64)[None, :]
        pa[r] = gg[r].sum(axis=1)
        pb[r] = (gg[r] * xh[r]).sum(axis=1)
    ckey = lambda e: (e.col0, e.cols)
    rkey = lambda e: (e.row0, e.rows)
    sa, sb = {}, {}
    for r in range(grid.world):
        if r not in sa:
            sa.update(_allreduce_distinct(fab, ex, row_g[r], ckey, pa))
            sb.update(_allreduce_distinct(fab, ex, row_g[r], ckey, pb))
    dXs, dg, db = {}, {}, {}
    for r in range(grid.world):
        rstd = saved[r][1]
        dXs[r] = rstd[:, None] * (gg[r] - sa[r][:, None] / H - xh[r] * sb[r][:, None] / H)
    # column partials: sum over the local rows, then over the distinct row blocks that share
    # these columns (replicated row blocks are counted once: take one holder per row block)
    pg = {r: (np.asarray(dYs[r], np.float64) * xh[r]).sum(axis=0) for r in range(grid.world)}
    pbeta = {r: np.asarray(dYs[r], np.float64).sum(axis=0) for r in range(grid.world)}
    for r in range(grid.world):
        if r not in dg:
            dg.update(_allreduce_distinct(fab, ex, col_g[r], rkey, pg))
            db.update(_allreduce_distinct(fab, ex, col_g[r], rkey, pbeta))
    return dXs, dg, db
