"""Solomonik-style 2.5D linear layer. TEST INFRASTRUCTURE ONLY.

P:L526 cites 2.5D matrix multiplication (Solomonik & Demmel): p = d q^2 processors as d
layers of a q x q grid, the operands REPLICATED on every layer, each layer doing 1/d of the
SUMMA steps, the layers' results combined over depth. This differs from the paper's own
(Colossal-AI) 2.5D, whose layers split the batch (a-8). Reading N5:

  layout   rank (dep, i, j) holds X[i,j] [M/q, K/q], W[i,j] [K/q, N/q], Y[i,j] [M/q, N/q] and
           bias block j, the same on every layer (replicas);
  steps    layer dep runs the SUMMA steps T_dep = [dep q/d, (dep+1) q/d)   (q % d == 0);
  fwd      Y_dep[i,j] = sum_{t in T_dep} X[i,t] W[t,j]  (row bcast of X[i,t] from column t,
           column bcast of W[t,j] from row t, inside the layer); Y = AR_depth(alpha Y_dep),
           bias added once (layer 0's partial);
  bwd dX   for k in T_dep: bcast W[k,j] down column j (root row k), P = dY[i,j] W[k,j]^T,
           reduce P along row i to column k -> dX[i,k] on layer dep; then every rank gets its
           dX[i,j] by a depth broadcast from layer j // (q/d);
  bwd dW   for k in T_dep: bcast X[i,k] along row i (root column k), P = X[i,k]^T dY[i,j],
           reduce along column j to row k -> dW[k,j]; depth broadcast from layer i // (q/d);
  db       colsum of dY[i,j], all-reduced along column j (dY is replicated over depth).

Every rank does 6 M K N / p flops (the work splits over depth). Volume (SPEC conventions,
elements): fwd (q-1)(S_x+S_w) + 2(d-1) S_y; bwd 2(q-1)(S_x+S_w) + (d-1)(S_x+S_w)
(closed_form_volume). Parity unpinned: nothing in the paper gives this scheme's numbers; the
pins are the dense definition, d = 1 == SUMMA bitwise, brute force and the ledger.
"""
from __future__ import annotations

import numpy as np

from .fabric import Fabric
from .grid import AX_25_DEP, AX_25_I, AX_25_J, Grid
from .shards import Extent, LayerSpec


def check(grid: Grid, spec: LayerSpec) -> None:
    if grid.mode != "2.5d":
        raise ValueError("Solomonik 2.5D runs on a 2.5D grid")
    q, d = grid.q, grid.d
    if q % d:
        raise ValueError(f"q = {q} not divisible by d = {d}")
    for v, what in ((spec.M, "M"), (spec.K, "K"), (spec.N, "N")):
        if v % q:
            raise ValueError(f"{what}={v} not divisible by {q}")


def extent(grid: Grid, spec: LayerSpec, rank: int, tensor: str) -> Extent:
    check(grid, spec)
    _, i, j = grid.coords(rank)
    q, M, K, N = grid.q, spec.M, spec.K, spec.N
    if tensor == "X":
        return Extent(i * M // q, M // q, j * K // q, K // q)
    if tensor == "W":
        return Extent(i * K // q, K // q, j * N // q, N // q)
    if tensor == "Y":
        return Extent(i * M // q, M // q, j * N // q, N // q)
    if tensor == "B":
        return Extent(0, 1, j * N // q, N // q)
    raise ValueError(tensor)


def shard(grid: Grid, spec: LayerSpec, G, tensor: str) -> dict:
    G2 = np.asarray(G)[None, :] if tensor == "B" else np.asarray(G)
    out = {}
    for r in range(grid.world):
        blk = extent(grid, spec, r, tensor).take(G2).copy()
        out[r] = blk[0] if tensor == "B" else blk
    return out


def gather_full(grid: Grid, spec: LayerSpec, shards: dict, tensor: str) -> np.ndarray:
    """Reassemble; every replica (one per layer) must agree exactly."""
    full = {"X": (spec.M, spec.K), "W": (spec.K, spec.N), "Y": (spec.M, spec.N), "B": (1, spec.N)}[tensor]
    G = np.full(full, np.nan)
    for r in range(grid.world):
        e = extent(grid, spec, r, tensor)
        blk = np.asarray(shards[r], dtype=np.float64)
        blk = blk[None, :] if tensor == "B" else blk
        if blk.shape != (e.rows, e.cols):
            raise ValueError(f"ShapeMismatch rank {r}: {blk.shape} vs {(e.rows, e.cols)}")
        view = G[e.row0:e.row0 + e.rows, e.col0:e.col0 + e.cols]
        have = ~np.isnan(view)
        if have.any() and not np.array_equal(view[have], blk[have]):
            raise AssertionError(f"replicas disagree at rank {r} for {tensor}")
        G[e.row0:e.row0 + e.rows, e.col0:e.col0 + e.cols] = blk
    if np.isnan(G).any():
        raise AssertionError(f"{tensor} not fully covered")
    return G[0] if tensor == "B" else G


def steps(q: int, d: int, dep: int) -> range:
    """T_dep: the SUMMA steps layer dep runs."""
    w = q // d
    return range(dep * w, (dep + 1) * w)


def _layer(grid: Grid, dep: int):
    """(rank -> (i, j)) for the ranks of layer dep, and that layer's row / column groups."""
    members = [r for r in range(grid.world) if grid.coords(r)[0] == dep]
    rows = [g for g in grid.groups_along(AX_25_J) if g[0] in members]   # fixed (dep, i)
    cols = [g for g in grid.groups_along(AX_25_I) if g[0] in members]   # fixed (dep, j)
    return members, rows, cols


def fwd(grid: Grid, X: dict, W: dict, b=None, alpha=1.0, fab: Fabric | None = None) -> dict:
    fab = fab or Fabric()
    q, d = grid.q, grid.d
    part = {}
    for dep in range(d):
        members, rows, cols = _layer(grid, dep)
        acc = {r: None for r in members}
        for t in steps(q, d, dep):
            xb, wb = {}, {}
            for g in rows:   # row i: root at column t
                xb.update(fab.broadcast(g, g[t], X[g[t]]))
            for g in cols:   # column j: root at row t
                wb.update(fab.broadcast(g, g[t], W[g[t]]))
            for r in members:
                prod = xb[r] @ wb[r]
                acc[r] = prod if acc[r] is None else acc[r] + prod
        for r in members:
            part[r] = alpha * acc[r]
            if b is not None and dep == 0:
                part[r] = part[r] + np.asarray(b[r], np.float64)[None, :]
    Y = {}
    for g in grid.groups_along(AX_25_DEP):
        Y.update(fab.all_reduce(g, {r: part[r] for r in g}))
    return Y


def bwd(grid: Grid, dY: dict, X: dict, W: dict, alpha=1.0, fab: Fabric | None = None):
    """Returns per-rank (dX, dW, db)."""
    fab = fab or Fabric()
    q, d = grid.q, grid.d
    w = q // d
    dX_own, dW_own = {}, {}
    for dep in range(d):
        members, rows, cols = _layer(grid, dep)
        for k in steps(q, d, dep):
            # dX[i,k] = sum_j dY[i,j] W[k,j]^T: W[k,j] down column j from row k, reduce along row i
            wb = {}
            for g in cols:
                wb.update(fab.broadcast(g, g[k], W[g[k]]))
            P = {r: alpha * (np.asarray(dY[r], np.float64) @ wb[r].T) for r in members}
            for g in rows:
                dX_own[g[k]] = fab.reduce(g, g[k], {r: P[r] for r in g})
            # dW[k,j] = sum_i X[i,k]^T dY[i,j]: X[i,k] along row i from column k, reduce down column j
            xb = {}
            for g in rows:
                xb.update(fab.broadcast(g, g[k], X[g[k]]))
            P = {r: alpha * (xb[r].T @ np.asarray(dY[r], np.float64)) for r in members}
            for g in cols:
                dW_own[g[k]] = fab.reduce(g, g[k], {r: P[r] for r in g})
    dX, dW = {}, {}
    for g in grid.groups_along(AX_25_DEP):    # fixed (i, j), layers ascending
        _, i, j = grid.coords(g[0])
        dX.update(fab.broadcast(g, g[j // w], dX_own[g[j // w]]))
        dW.update(fab.broadcast(g, g[i // w], dW_own[g[i // w]]))
    db = {}
    for g in grid.groups_along(AX_25_I):      # fixed (dep, j): column sums, all-reduced
        db.update(fab.all_reduce(g, {r: np.asarray(dY[r], np.float64).sum(axis=0) for r in g}))
    return dX, dW, db


def closed_form_volume(grid: Grid, spec: LayerSpec) -> dict:
    """Elements moved (SPEC conventions) by fwd and bwd of one layer."""
    q, d = grid.q, grid.d
    Sx, Sw, Sy = spec.M * spec.K, spec.K * spec.N, spec.M * spec.N
    return {"fwd": (q - 1) * (Sx + Sw) + 2 * (d - 1) * Sy,
            "bwd": 2 * (q - 1) * (Sx + Sw) + (d - 1) * (Sx + Sw)}
