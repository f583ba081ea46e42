"""Cannon's algorithm for the 2D forward product (NEXT-4 variant). TEST INFRASTRUCTURE ONLY.

P:L524: "2D tensor parallelism relies on the SUMMA and Cannon matrix multiplication
algorithm" (Cannon 1969). Same q x q grid and the same shard layout as the SUMMA schedule
(shards.extent, 2D): rank (i,j) holds X[i,j], W[i,j] and produces Y[i,j] = sum_t
X[i,t] W[t,j]. Cannon's order, per rank:

  skew:    row i of X shifts left by i   -> rank (i,j) holds X[i, (i+j) mod q]
           column j of W shifts up by j  -> rank (i,j) holds W[(i+j) mod q, j]
  q steps: Y[i,j] += X_held . W_held; then X shifts left by 1 along the row and W up by 1
           along the column (the last step needs no shift).

"Shift left by s along a line" = every member receives the block of the member s positions
after it (mod q). Each shift sends one block per member (ledger "shift"): the skew moves the
blocks of the q-1 rows / columns with a non-zero offset, then q-1 unit shifts move all.
"""
from __future__ import annotations

import numpy as np

from .fabric import Fabric
from .grid import AX_2D_I, AX_2D_J, Grid


def _shift(fab: Fabric, group, held: dict, s: int) -> dict:
    """Member at position p receives the block of position (p + s) mod g."""
    g = len(group)
    if s % g == 0:
        return dict(held)
    out = {}
    for p, r in enumerate(group):
        src = group[(p + s) % g]
        out[r] = held[src]
        fab.ledger.add("shift", tuple(group), src, r, int(np.size(held[src])))
    return out


def cannon_fwd(grid: Grid, X: dict, W: dict, b=None, alpha=1.0, fab=None):
    """Per-rank Y = alpha sum_t X[i,t] W[t,j] (+ b) with Cannon's schedule."""
    fab = fab or Fabric()
    q = grid.q
    rows = grid.groups_along(AX_2D_J)   # fixed i, j varies (ascending j)
    cols = grid.groups_along(AX_2D_I)   # fixed j, i varies (ascending i)
    Xh = {r: np.asarray(X[r], np.float64) for r in X}
    Wh = {r: np.asarray(W[r], np.float64) for r in W}
    for g in rows:                       # skew X: row i left by i
        i = grid.coords(g[0])[0]
        Xh.update(_shift(fab, g, Xh, i))
    for g in cols:                       # skew W: column j up by j
        j = grid.coords(g[0])[1]
        Wh.update(_shift(fab, g, Wh, j))
    acc = {r: None for r in X}
    for t in range(q):
        for r in acc:
            prod = Xh[r] @ Wh[r]
            acc[r] = prod if acc[r] is None else acc[r] + prod
        if t + 1 < q:
            for g in rows:
                Xh.update(_shift(fab, g, Xh, 1))
            for g in cols:
                Wh.update(_shift(fab, g, Wh, 1))
    Y = {}
    for r in acc:
        Y[r] = alpha * acc[r]
        if b is not None:
            Y[r] = Y[r] + np.asarray(b[r], np.float64)[None, :]
    return Y


def cannon_bwd(grid: Grid, dY: dict, X: dict, W: dict, alpha=1.0, fab=None):
    """Per-rank (dX, dW) of the 2D layer with Cannon's schedule, the accumulator moving
    ("SUMMA and Cannon"; the paper states the forward; the backward products are the same
    algorithm with one operand and the partial sums circulating - reading N7):

      dX[i,k] = sum_j dY[i,j] W[k,j]^T : dY stationary; W skewed up by j along column j, then
        shifted up by 1 per step; at step t rank (i,j) adds dY[i,j] W[(i+j+t) mod q, j]^T to
        the accumulator of dX[i, (i+j+t) mod q] it holds, then every accumulator moves left by
        1 along the row; after q steps the one for dX[i,k] sits at column k - i and a final
        shift by -i along row i delivers it to its owner (i,k).
      dW[k,j] = sum_i X[i,k]^T dY[i,j] : dY stationary; X skewed left by i along row i, then
        shifted left by 1 per step; rank (i,j) adds X[i,(i+j+t) mod q]^T dY[i,j] to the
        accumulator of dW[(i+j+t) mod q, j]; accumulators move up by 1 along the column; a
        final shift by -j along column j delivers dW[k,j] to (k,j).
    Accumulators are fp64 here (the GPU carries fp32 partials on the wire)."""
    fab = fab or Fabric()
    q = grid.q
    rows = grid.groups_along(AX_2D_J)
    cols = grid.groups_along(AX_2D_I)
    dYh = {r: np.asarray(dY[r], np.float64) for r in dY}
    # ---- dX (ABT)
    Wh = {r: np.asarray(W[r], np.float64) for r in W}
    for g in cols:                       # skew W: column j up by j
        Wh.update(_shift(fab, g, Wh, grid.coords(g[0])[1]))
    acc = {r: None for r in dY}
    for t in range(q):
        for r in acc:
            part = dYh[r] @ Wh[r].T
            acc[r] = part if acc[r] is None else acc[r] + part
        for g in rows:                   # accumulators one column to the left
            acc.update(_shift(fab, g, acc, 1))
        if t + 1 < q:
            for g in cols:
                Wh.update(_shift(fab, g, Wh, 1))
    for g in rows:                       # deliver: row i shifts by -i
        acc.update(_shift(fab, g, acc, -grid.coords(g[0])[0]))
    dX = {r: alpha * acc[r] for r in acc}
    # ---- dW (ATB)
    Xh = {r: np.asarray(X[r], np.float64) for r in X}
    for g in rows:                       # skew X: row i left by i
        Xh.update(_shift(fab, g, Xh, grid.coords(g[0])[0]))
    acc = {r: None for r in dY}
    for t in range(q):
        for r in acc:
            part = Xh[r].T @ dYh[r]
            acc[r] = part if acc[r] is None else acc[r] + part
        for g in cols:                   # accumulators one row up
            acc.update(_shift(fab, g, acc, 1))
        if t + 1 < q:
            for g in rows:
                Xh.update(_shift(fab, g, Xh, 1))
    for g in cols:                       # deliver: column j shifts by -j
        acc.update(_shift(fab, g, acc, -grid.coords(g[0])[1]))
    dW = {r: alpha * acc[r] for r in acc}
    return dX, dW
