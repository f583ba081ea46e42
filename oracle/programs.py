"""Rank-by-rank fp64 programs of every TP mode, forward and backward. TEST INFRASTRUCTURE ONLY.

Each function simulates all ranks of the grid in lock-step over the Fabric
(simulated collectives + ledger) and returns per-rank outputs (dict rank->array).
The loops follow SURVEY.md 8(a), which restates the paper:

  1D col  (a-3)  P:L486-488: Y_r = X.W_r, no forward comm; dX = AR_p(dY_r.W_r^T).
  1D row  (a-4)  P:L488 "An all-reduce operation can be applied on the partial
                 result": Y = AR_p(X_r.W_r); dX_r = dY.W_r^T, no comm.
  2D      (a-5..a-7) P:L524 SUMMA: for t: bcast X[i,t] along row i, bcast W[t,j]
                 along column j, Y[i,j] += X[i,t].W[t,j]. Backward = two more
                 SUMMA products (Table tp-comm-vol factor 3):
                 dX[i,k] = reduce_row( dY[i,j].W[k,j]^T )  ("ABT"),
                 dW[k,j] = reduce_col( X[i,k]^T.dY[i,j] )  ("ATB").
  2.5D    (a-8)  P:L526: each depth plane runs the 2D program on its batch
                 slice; the depth axis then sums dW (all-reduce, replicated W)
                 or all-gathers W before / reduce-scatters dW after (depth-sharded W).
  3D      (a-9, a-10) P:L528: AG(X) over one axis, AG(W) over another, local
                 product, RS(Y) over the third; backward AG(dY), RS(dX), RS(dW).

Alpha scales the product (Y = alpha*X.W + b); bias (reading A16) is added once,
on the rank whose partial is summed first, or after the all-reduce.
"""
from __future__ import annotations

import numpy as np

from .fabric import Fabric
from .grid import (AX_25_DEP, AX_25_I, AX_25_J, AX_2D_I, AX_2D_J, AX_3D_A, AX_3D_B,
                   AX_3D_C, Grid)
from .shards import LayerSpec, check_divisible


def _mm(A, B):
    return np.asarray(A, np.float64) @ np.asarray(B, np.float64)


def _groups(grid: Grid, axis: int, ranks=None):
    return grid.groups_along(axis) if ranks is None else \
        [g for g in grid.groups_along(axis) if g[0] in ranks]


# ----------------------------------------------------------------------------- 1D

def fwd_1d(grid, spec, X, W, b=None, alpha=1.0, fab=None):
    fab = fab or Fabric()
    world = list(range(grid.world))
    if spec.split_1d == "col":
        Y = {}
        for r in world:
            Y[r] = alpha * _mm(X[r], W[r])
            if b is not None:
                Y[r] = Y[r] + np.asarray(b[r], np.float64)[None, :]
        return Y, {}
    P = {}
    for r in world:
        P[r] = alpha * _mm(X[r], W[r])
        if b is not None and r == 0:
            P[r] = P[r] + np.asarray(b[r], np.float64)[None, :]
    return fab.all_reduce(world, P), {}


def bwd_1d(grid, spec, dY, X, W, alpha=1.0, fab=None, saved=None):
    fab = fab or Fabric()
    world = list(range(grid.world))
    dW = {r: alpha * _mm(np.asarray(X[r]).T, dY[r]) for r in world}
    db = {r: np.asarray(dY[r], np.float64).sum(axis=0) for r in world}
    if spec.split_1d == "col":
        P = {r: alpha * _mm(dY[r], np.asarray(W[r]).T) for r in world}
        dX = fab.all_reduce(world, P)
    else:
        dX = {r: alpha * _mm(dY[r], np.asarray(W[r]).T) for r in world}
    return dX, dW, db


# ----------------------------------------------------------------------------- 2D

def _summa_fwd(grid, ranks, ax_i, ax_j, X, W, fab):
    """Y[i,j] = sum_t X[i,t].W[t,j] over the q x q sub-grid `ranks` (SUMMA "AB")."""
    q = grid.dims[ax_j]
    acc = {r: None for r in ranks}
    rows = [g for g in grid.groups_along(ax_j) if g[0] in ranks]   # fixed i, j varies
    cols = [g for g in grid.groups_along(ax_i) if g[0] in ranks]   # fixed j, i varies
    for t in range(q):
        Xt, Wt = {}, {}
        for g in rows:
            Xt.update(fab.broadcast(g, g[t], X[g[t]]))       # root = column t of row i
        for g in cols:
            Wt.update(fab.broadcast(g, g[t], W[g[t]]))       # root = row t of column j
        for r in ranks:
            prod = _mm(Xt[r], Wt[r])
            acc[r] = prod if acc[r] is None else acc[r] + prod
    return acc


def _summa_abt(grid, ranks, ax_i, ax_j, dY, W, alpha, fab):
    """dX[i,k] = sum_j dY[i,j].W[k,j]^T: bcast W down columns, reduce along rows."""
    q = grid.dims[ax_j]
    rows = [g for g in grid.groups_along(ax_j) if g[0] in ranks]
    cols = [g for g in grid.groups_along(ax_i) if g[0] in ranks]
    dX = {}
    for k in range(q):
        Wk = {}
        for g in cols:
            Wk.update(fab.broadcast(g, g[k], W[g[k]]))
        P = {r: alpha * _mm(dY[r], Wk[r].T) for r in ranks}
        for g in rows:
            dX[g[k]] = fab.reduce(g, g[k], {r: P[r] for r in g})
    return dX


def _summa_atb(grid, ranks, ax_i, ax_j, X, dY, alpha, fab):
    """dW[k,j] = sum_i X[i,k]^T.dY[i,j]: bcast X along rows, reduce down columns."""
    q = grid.dims[ax_j]
    rows = [g for g in grid.groups_along(ax_j) if g[0] in ranks]
    cols = [g for g in grid.groups_along(ax_i) if g[0] in ranks]
    dW = {}
    for k in range(q):
        Xk = {}
        for g in rows:
            Xk.update(fab.broadcast(g, g[k], X[g[k]]))
        P = {r: alpha * _mm(np.asarray(Xk[r]).T, dY[r]) for r in ranks}
        for g in cols:
            dW[g[k]] = fab.reduce(g, g[k], {r: P[r] for r in g})
    return dW


def fwd_2d(grid, spec, X, W, b=None, alpha=1.0, fab=None):
    fab = fab or Fabric()
    ranks = list(range(grid.world))
    acc = _summa_fwd(grid, ranks, AX_2D_I, AX_2D_J, X, W, fab)
    Y = {}
    for r in ranks:
        Y[r] = alpha * acc[r]
        if b is not None:
            Y[r] = Y[r] + np.asarray(b[r], np.float64)[None, :]
    return Y, {}


def bwd_2d(grid, spec, dY, X, W, alpha=1.0, fab=None, saved=None):
    fab = fab or Fabric()
    ranks = list(range(grid.world))
    dX = _summa_abt(grid, ranks, AX_2D_I, AX_2D_J, dY, W, alpha, fab)
    dW = _summa_atb(grid, ranks, AX_2D_I, AX_2D_J, X, dY, alpha, fab)
    cs = {r: np.asarray(dY[r], np.float64).sum(axis=0) for r in ranks}
    db = {}
    for g in grid.groups_along(AX_2D_I):                  # ranks sharing column block j
        db.update(fab.all_reduce(g, {r: cs[r] for r in g}))
    return dX, dW, db


# ----------------------------------------------------------------------------- 2.5D

def _planes(grid):
    q2 = grid.q * grid.q
    return [list(range(dep * q2, (dep + 1) * q2)) for dep in range(grid.d)]


def fwd_25d(grid, spec, X, W, b=None, alpha=1.0, fab=None):
    fab = fab or Fabric()
    saved = {}
    if spec.w_depth_sharded:
        Wfull = {}
        for g in grid.groups_along(AX_25_DEP):
            Wfull.update(fab.all_gather(g, {r: W[r] for r in g}, axis=0))
        saved["W"] = Wfull
        W = Wfull
    Y = {}
    for plane in _planes(grid):
        acc = _summa_fwd(grid, plane, AX_25_I, AX_25_J, X, W, fab)
        for r in plane:
            Y[r] = alpha * acc[r]
            if b is not None:
                Y[r] = Y[r] + np.asarray(b[r], np.float64)[None, :]
    return Y, saved


def bwd_25d(grid, spec, dY, X, W, alpha=1.0, fab=None, saved=None):
    fab = fab or Fabric()
    if spec.w_depth_sharded:
        W = saved["W"]          # gathered in forward (the SAVE contract)
    dX, dWp = {}, {}
    for plane in _planes(grid):
        dX.update(_summa_abt(grid, plane, AX_25_I, AX_25_J, dY, W, alpha, fab))
        dWp.update(_summa_atb(grid, plane, AX_25_I, AX_25_J, X, dY, alpha, fab))
    dW = {}
    for g in grid.groups_along(AX_25_DEP):
        parts = {r: dWp[r] for r in g}
        if spec.w_depth_sharded:
            dW.update(fab.reduce_scatter(g, parts, axis=0))
        else:
            dW.update(fab.all_reduce(g, parts))
    cs = {r: np.asarray(dY[r], np.float64).sum(axis=0) for r in range(grid.world)}
    db = {}
    for g in grid.groups_along(AX_25_I):              # within plane, same column block
        db.update(fab.all_reduce(g, {r: cs[r] for r in g}))
    out = {}
    for g in grid.groups_along(AX_25_DEP):
        out.update(fab.all_reduce(g, {r: db[r] for r in g}))
    return dX, dW, out


# ----------------------------------------------------------------------------- 3D

def _axes_3d(parity):
    """(X-gather axis, W-gather axis, Y-scatter axis)."""
    return (AX_3D_C, AX_3D_A, AX_3D_B) if parity == 0 else (AX_3D_B, AX_3D_A, AX_3D_C)


def fwd_3d(grid, spec, X, W, b=None, alpha=1.0, fab=None):
    fab = fab or Fabric()
    ax_x, ax_w, ax_y = _axes_3d(spec.parity)
    Xg, Wg = {}, {}
    for g in grid.groups_along(ax_x):
        Xg.update(fab.all_gather(g, {r: X[r] for r in g}, axis=0))
    for g in grid.groups_along(ax_w):
        Wg.update(fab.all_gather(g, {r: W[r] for r in g}, axis=0))
    P = {}
    for r in range(grid.world):
        P[r] = alpha * _mm(Xg[r], Wg[r])
        if b is not None and grid.coords(r)[ax_y] == 0:
            P[r] = P[r] + np.asarray(b[r], np.float64)[None, :]
    Y = {}
    for g in grid.groups_along(ax_y):
        Y.update(fab.reduce_scatter(g, {r: P[r] for r in g}, axis=0))
    return Y, {"X": Xg, "W": Wg}


def bwd_3d(grid, spec, dY, X, W, alpha=1.0, fab=None, saved=None):
    fab = fab or Fabric()
    ax_x, ax_w, ax_y = _axes_3d(spec.parity)
    Xg, Wg = saved["X"], saved["W"]        # reused from forward: no re-gather (reading A10)
    dYg = {}
    for g in grid.groups_along(ax_y):
        dYg.update(fab.all_gather(g, {r: dY[r] for r in g}, axis=0))
    Px = {r: alpha * _mm(dYg[r], np.asarray(Wg[r]).T) for r in range(grid.world)}
    Pw = {r: alpha * _mm(np.asarray(Xg[r]).T, dYg[r]) for r in range(grid.world)}
    dX, dW = {}, {}
    for g in grid.groups_along(ax_x):
        dX.update(fab.reduce_scatter(g, {r: Px[r] for r in g}, axis=0))
    for g in grid.groups_along(ax_w):
        dW.update(fab.reduce_scatter(g, {r: Pw[r] for r in g}, axis=0))
    cs = {r: dYg[r].sum(axis=0) for r in range(grid.world)}
    db = {}
    for g in grid.groups_along(AX_3D_A):
        db.update(fab.all_reduce(g, {r: cs[r] for r in g}))
    return dX, dW, db


# ----------------------------------------------------------------------------- dispatch

_FWD = {"1d": fwd_1d, "2d": fwd_2d, "2.5d": fwd_25d, "3d": fwd_3d}
_BWD = {"1d": bwd_1d, "2d": bwd_2d, "2.5d": bwd_25d, "3d": bwd_3d}


def layer_fwd(grid: Grid, spec: LayerSpec, X, W, b=None, alpha=1.0, fab=None):
    """Per-rank forward. Returns (Y shards, saved) where saved holds gathered operands."""
    check_divisible(grid, spec)
    return _FWD[grid.mode](grid, spec, X, W, b, alpha, fab)


def layer_bwd(grid: Grid, spec: LayerSpec, dY, X, W, alpha=1.0, fab=None, saved=None):
    """Per-rank backward. Returns (dX, dW, db) shards."""
    check_divisible(grid, spec)
    return _BWD[grid.mode](grid, spec, dY, X, W, alpha, fab, saved)


def mlp2_specs(grid: Grid, M: int, H: int, F: int | None = None, w_depth_sharded=False):
    """Layer specs of the two-linear-layer model whose layer-1 Y layout IS layer-2's X
    layout: 1D col then row (P:L488 Megatron pairing), 3D parity 0 then 1 (reading A9)."""
    F = H if F is None else F
    s1 = LayerSpec(M, H, F, split_1d="col", parity=0, w_depth_sharded=w_depth_sharded)
    s2 = LayerSpec(M, F, H, split_1d="row", parity=1, w_depth_sharded=w_depth_sharded)
    return s1, s2
