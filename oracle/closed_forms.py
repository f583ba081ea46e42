"""Closed forms: the paper's communication table, our schedule's exact counts, memory.

TEST INFRASTRUCTURE ONLY.

paper_comm_volume   Table tp-comm-vol, evaluated verbatim:
                      1D   2(p-1) S_x
                      2D   3(j-1) (S_x + S_w)
                      2.5D 3(k-1) (S_x/d + S_w)
                      3D   2(l-1)/l (S_x + S_w + S_y)
                    (P:L391-403 notation; S_y = S_x for square W, reading A1).
counted_volume      what the schedules of programs.py move, in the same element
                    units and SPEC's collective conventions (fabric.py), per
                    single linear layer, bias-free. Readings A3 (1D is per layer),
                    A4 (2D exact), A10 (3D moves each tensor twice -> ratio l),
                    A11 (2.5D Table row is per plane; depth term extra).
memory_per_rank     at-rest elements of X, W, Y shards (P:L524-528 shard shapes)
                    and the two-layer model totals compared with the paper's
                    range-test percentages.
"""
from __future__ import annotations

from fractions import Fraction


def paper_comm_volume(mode: str, S_x, S_w, S_y=None, p=None, j=None, k=None, d=None, l=None):
    S_y = S_x if S_y is None else S_y
    if mode == "1d":
        return 2 * (p - 1) * S_x
    if mode == "2d":
        return 3 * (j - 1) * (S_x + S_w)
    if mode == "2.5d":
        return 3 * (k - 1) * (Fraction(S_x, d) + S_w)
    if mode == "3d":
        return Fraction(2 * (l - 1), l) * (S_x + S_w + S_y)
    raise ValueError(mode)


def counted_volume(mode: str, M: int, K: int, N: int, p: int = 1, q: int = 1, d: int = 1,
                   split_1d: str = "col", part: str = "fwd+bwd") -> int:
    """Elements our schedule moves for one layer (aggregate, SPEC conventions)."""
    Sx, Sw, Sy = M * K, K * N, M * N
    if mode == "1d":
        fwd = 0 if split_1d == "col" else 2 * (p - 1) * Sy
        bwd = 2 * (p - 1) * Sx if split_1d == "col" else 0
    elif mode == "2d":
        fwd = (q - 1) * (Sx + Sw)
        bwd = 2 * (q - 1) * (Sx + Sw)
    elif mode == "2.5d":
        # d planes of SUMMA on Sx/d rows + depth AR of dW (or AG W + RS dW): 2(d-1) Sw
        fwd = d * (q - 1) * (Sx // d + Sw)
        bwd = 2 * d * (q - 1) * (Sx // d + Sw)
        depth = 2 * (d - 1) * Sw
        return {"fwd": fwd, "bwd": bwd, "depth": depth,
                "fwd+bwd": fwd + bwd + depth}[part]
    elif mode == "3d":
        fwd = (q - 1) * (Sx + Sw + Sy)
        bwd = (q - 1) * (Sx + Sw + Sy)
    else:
        raise ValueError(mode)
    return {"fwd": fwd, "bwd": bwd, "fwd+bwd": fwd + bwd}[part]


def memory_per_rank(mode: str, M: int, K: int, N: int, p: int, q: int = 1, d: int = 1,
                    split_1d: str = "col", w_depth_sharded: bool = False) -> dict:
    """At-rest elements per rank of one layer's X, W, Y shards."""
    Sx, Sw, Sy = M * K, K * N, M * N
    if mode == "1d":
        if split_1d == "col":
            return {"X": Sx, "W": Sw // p, "Y": Sy // p}
        return {"X": Sx // p, "W": Sw // p, "Y": Sy}
    if mode in ("2d", "3d"):
        return {"X": Sx // p, "W": Sw // p, "Y": Sy // p}
    if mode == "2.5d":
        return {"X": Sx // p, "W": Sw // p if w_depth_sharded else Sw // (q * q), "Y": Sy // p}
    raise ValueError(mode)


def mlp2_memory(mode: str, M: int, h: int, p: int, q: int = 1, d: int = 1,
                w_depth_sharded: bool = False) -> Fraction:
    """Per-rank at-rest elements of the two square layers' X, Y1, Y2, W1, W2."""
    a, w = M * h, h * h
    if mode == "1d":       # X and Y2 replicated, Y1 split by columns, W split
        return Fraction(2 * a) + Fraction(a, p) + Fraction(2 * w, p)
    if mode in ("2d", "3d"):
        return Fraction(3 * a, p) + Fraction(2 * w, p)
    if mode == "2.5d":
        wr = Fraction(w, p) if w_depth_sharded else Fraction(w, q * q)
        return Fraction(3 * a, p) + 2 * wr
    raise ValueError(mode)


def memory_reduction_vs_1d(mode: str, M: int, h: int, p: int, q: int = 1, d: int = 1) -> float:
    """1 - mem(mode)/mem(1D), the quantity the paper reports in P:L81."""
    return float(1 - mlp2_memory(mode, M, h, p, q, d) / mlp2_memory("1d", M, h, p))
