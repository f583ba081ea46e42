"""Per-rank shard extents of X [M,K], W [K,N], Y [M,N] and bias [N]. TEST INFRASTRUCTURE ONLY.

Passages:
  1D  P:L486-488: column-parallel splits W by columns (X replicated, Y split by
      columns); row-parallel splits W by rows (X split by columns, Y replicated
      after the all-reduce "on the partial result").
  2D  P:L524 "a tensor of shape [P, Q] will be partitioned into a chunk tensor of
      shape [P/sqrt(N), Q/sqrt(N)]" on a row-major q x q grid.
  2.5D P:L526 "partitions the matrix 3 times": activations split by depth along
      the batch rows, then q x q within the plane; W per plane q x q,
      replicated over depth (reading A6) or additionally split over depth
      (W25_DEPTH_SHARDED, the north star's 1/p memory).
  3D  P:L528 "[P/cbrt(N)^2, Q/cbrt(N)]": the first dim split twice, the last once.
      Axis roles per SURVEY 8(a) a-9 (reading A9): parity 0 gathers X over c, W
      over a, scatters Y over b; parity 1 swaps b and c so that Y(parity 0) is
      exactly X(parity 1).
Gradients take the layout of their tensor (dX ~ X, dW ~ W, dY ~ Y, db ~ bias).
Divisibility is a hard precondition, no padding (reading A15).
"""
from __future__ import annotations

from dataclasses import dataclass

from .grid import Grid


class IndivisibleDim(ValueError):
    """A global dim is not divisible by the split the mode needs."""


@dataclass(frozen=True)
class LayerSpec:
    M: int
    K: int
    N: int
    split_1d: str = "col"      # "col" | "row"
    parity: int = 0            # 3D layer parity
    w_depth_sharded: bool = False  # 2.5D weight layout


@dataclass(frozen=True)
class Extent:
    row0: int
    rows: int
    col0: int
    cols: int

    def take(self, G):
        return G[self.row0:self.row0 + self.rows, self.col0:self.col0 + self.cols]


def _div(a: int, b: int, what: str) -> int:
    if b <= 0 or a % b:
        raise IndivisibleDim(f"{what}: {a} not divisible by {b}")
    return a // b


def check_divisible(grid: Grid, spec: LayerSpec) -> None:
    M, K, N = spec.M, spec.K, spec.N
    p, q = grid.world, grid.q
    if grid.mode == "1d":
        if spec.split_1d == "col":
            _div(N, p, "1D col: N")
        elif spec.split_1d == "row":
            _div(K, p, "1D row: K")
        else:
            raise ValueError(spec.split_1d)
    elif grid.mode == "2d":
        _div(M, q, "M"); _div(K, q, "K"); _div(N, q, "N")
    elif grid.mode == "2.5d":
        d = grid.d
        _div(M, d * q, "M"); _div(N, q, "N")
        _div(K, q * d if spec.w_depth_sharded else q, "K")
    elif grid.mode == "3d":
        _div(M, q * q, "M"); _div(K, q * q, "K"); _div(N, q, "N")


def extent(grid: Grid, spec: LayerSpec, rank: int, tensor: str) -> Extent:
    """Global block (row0, rows, col0, cols) of `tensor` in {"X","W","Y","B"} held by `rank`."""
    check_divisible(grid, spec)
    M, K, N = spec.M, spec.K, spec.N
    c = grid.coords(rank)
    full = {"X": (M, K), "W": (K, N), "Y": (M, N), "B": (1, N)}[tensor]
    if grid.mode == "1d":
        (r,), p = c, grid.world
        if spec.split_1d == "col":
            if tensor == "X":
                return Extent(0, M, 0, K)
            if tensor == "W":
                return Extent(0, K, r * N // p, N // p)
            if tensor == "Y":
                return Extent(0, M, r * N // p, N // p)
            return Extent(0, 1, r * N // p, N // p)
        if tensor == "X":
            return Extent(0, M, r * K // p, K // p)
        if tensor == "W":
            return Extent(r * K // p, K // p, 0, N)
        return Extent(0, full[0], 0, full[1])          # Y, B replicated
    if grid.mode == "2d":
        i, j = c
        q = grid.q
        if tensor == "X":
            return Extent(i * M // q, M // q, j * K // q, K // q)
        if tensor == "W":
            return Extent(i * K // q, K // q, j * N // q, N // q)
        if tensor == "Y":
            return Extent(i * M // q, M // q, j * N // q, N // q)
        return Extent(0, 1, j * N // q, N // q)
    if grid.mode == "2.5d":
        dep, i, j = c
        q, d = grid.q, grid.d
        mb = M // (d * q)
        if tensor == "X":
            return Extent((dep * q + i) * mb, mb, j * K // q, K // q)
        if tensor == "W":
            if spec.w_depth_sharded:
                h = K // (q * d)
                return Extent(i * K // q + dep * h, h, j * N // q, N // q)
            return Extent(i * K // q, K // q, j * N // q, N // q)
        if tensor == "Y":
            return Extent((dep * q + i) * mb, mb, j * N // q, N // q)
        return Extent(0, 1, j * N // q, N // q)
    if grid.mode == "3d":
        a, b, cc = c
        l = grid.q
        if spec.parity == 1:
            b, cc = cc, b      # parity 1: the roles of axes b and c swap
        mb, kb = M // (l * l), K // (l * l)
        if tensor == "X":
            return Extent((a * l + cc) * mb, mb, b * K // l, K // l)
        if tensor == "W":
            return Extent((b * l + a) * kb, kb, cc * N // l, N // l)
        if tensor == "Y":
            return Extent((a * l + b) * mb, mb, cc * N // l, N // l)
        return Extent(0, 1, cc * N // l, N // l)
    raise ValueError(grid.mode)


def shard(grid: Grid, spec: LayerSpec, G, tensor: str) -> dict:
    """rank -> copy of its block of the global tensor G (bias given as 1-D [N])."""
    import numpy as np
    G2 = np.asarray(G)[None, :] if tensor == "B" else np.asarray(G)
    out = {}
    for r in range(grid.world):
        blk = extent(grid, spec, r, tensor).take(G2).copy()
        out[r] = blk[0] if tensor == "B" else blk
    return out


def gather_full(grid: Grid, spec: LayerSpec, shards: dict, tensor: str, check_replicas=True):
    """S:L321 gather_full: reassemble the global tensor; replicas must agree exactly."""
    import numpy as np
    full = {"X": (spec.M, spec.K), "W": (spec.K, spec.N), "Y": (spec.M, spec.N), "B": (1, spec.N)}[tensor]
    G = np.full(full, np.nan)
    for r in range(grid.world):
        e = extent(grid, spec, r, tensor)
        blk = np.asarray(shards[r], dtype=np.float64)
        blk = blk[None, :] if tensor == "B" else blk
        if blk.shape != (e.rows, e.cols):
            raise ValueError(f"ShapeMismatch rank {r}: {blk.shape} vs {(e.rows, e.cols)}")
        view = G[e.row0:e.row0 + e.rows, e.col0:e.col0 + e.cols]
        if check_replicas and not np.all(np.isnan(view)):
            have = ~np.isnan(view)
            if not np.array_equal(view[have], blk[have]):
                raise AssertionError(f"replicas disagree at rank {r} for {tensor}")
        G[e.row0:e.row0 + e.rows, e.col0:e.col0 + e.cols] = blk
    if np.isnan(G).any():
        raise AssertionError(f"{tensor} not fully covered")
    return G[0] if tensor == "B" else G
