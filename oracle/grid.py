"""Processor grids and per-axis groups. TEST INFRASTRUCTURE ONLY.

P:L530 "1D method can work with any number of GPUs while 2D, 2.5D and 3D
methods require the n^2, a*n^2, and n^3 GPUs respectively". P:L393-398 name the
sides: j (2D, p = j^2), k and d (2.5D, p = d*k^2), l (3D, p = l^3). P:L526 "S can
be calculated if D is given by the user" - depth is an input.
P:L413 "collective communication only involve the nodes in one row or one
column" - groups are the lines of the grid along one axis.

Readings: row-major rank order; 2.5D dims [depth, row, col]
with depth outermost (reading A7); 3D rank = a*l^2 + b*l + c (reading A9);
no silent fallback to 1D: a bad factorisation is ConstraintViolation.
Groups list their members by ascending coordinate along the axis.
"""
from __future__ import annotations

from dataclasses import dataclass


class ConstraintViolation(ValueError):
    """p does not factor as the mode requires."""


MODES = ("1d", "2d", "2.5d", "3d")


def _iroot(p: int, e: int) -> int | None:
    r = round(p ** (1.0 / e))
    for c in (r - 1, r, r + 1):
        if c >= 1 and c ** e == p:
            return c
    return None


@dataclass(frozen=True)
class Grid:
    mode: str
    world: int
    dims: tuple  # sizes of the coordinate axes

    @property
    def q(self) -> int:
        """Side of the square (2D j, 2.5D k) or cube (3D l); p for 1D."""
        return self.dims[-1]

    @property
    def d(self) -> int:
        return self.dims[0] if self.mode == "2.5d" else 1

    def coords(self, rank: int) -> tuple:
        if not 0 <= rank < self.world:
            raise ValueError("UnknownRank")
        out = []
        for size in reversed(self.dims):
            out.append(rank % size)
            rank //= size
        return tuple(reversed(out))

    def rank_of(self, coords) -> int:
        r = 0
        for c, size in zip(coords, self.dims):
            if not 0 <= c < size:
                raise ValueError("coordinate out of range")
            r = r * size + c
        return r

    def group(self, rank: int, axis: int) -> list:
        """Members of `rank`'s line along `axis` (that coordinate varies), ascending."""
        if not 0 <= axis < len(self.dims):
            raise ValueError("UnknownAxis")
        c = list(self.coords(rank))
        members = []
        for v in range(self.dims[axis]):
            c[axis] = v
            members.append(self.rank_of(c))
        return members

    def groups_along(self, axis: int) -> list:
        seen, out = set(), []
        for r in range(self.world):
            g = tuple(self.group(r, axis))
            if g not in seen:
                seen.add(g)
                out.append(list(g))
        return out


def build_grid(mode: str, world: int, depth: int = 1) -> Grid:
    """S:L41 build_mesh. 1D: [p]; 2D: [j, j]; 2.5D: [d, k, k]; 3D: [l, l, l]."""
    if world < 1:
        raise ConstraintViolation("world_size must be >= 1")
    if mode == "1d":
        return Grid(mode, world, (world,))
    if mode == "2d":
        j = _iroot(world, 2)
        if j is None:
            raise ConstraintViolation(f"2D needs p = j^2, got {world}")
        return Grid(mode, world, (j, j))
    if mode == "2.5d":
        if depth < 1 or world % depth:
            raise ConstraintViolation(f"2.5D needs p = d*k^2, got p={world}, d={depth}")
        k = _iroot(world // depth, 2)
        if k is None:
            raise ConstraintViolation(f"2.5D needs p = d*k^2, got p={world}, d={depth}")
        return Grid(mode, world, (depth, k, k))
    if mode == "3d":
        l = _iroot(world, 3)
        if l is None:
            raise ConstraintViolation(f"3D needs p = l^3, got {world}")
        return Grid(mode, world, (l, l, l))
    raise ValueError(f"unknown mode {mode}")


# Named axes (index into coords) used by the rank programs.
AX_2D_I, AX_2D_J = 0, 1            # group along J = "row i" group; along I = "column j" group
AX_25_DEP, AX_25_I, AX_25_J = 0, 1, 2
AX_3D_A, AX_3D_B, AX_3D_C = 0, 1, 2
