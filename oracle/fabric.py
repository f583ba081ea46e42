"""Simulated collectives on per-rank fp64 buffers, with an element ledger. TEST INFRASTRUCTURE ONLY.

Conventions follow SPEC.md's comm module (its accounting is the paper-facing
definition of "communication volume", Table tp-comm-vol header P:L370 "Total
Communication Volume / number of elements transferred"):
  broadcast       root sends m to each of the g-1 others        -> (g-1)*m
  reduce          each non-root sends its m to the root          -> (g-1)*m   (reading; mirror of bcast)
  all_reduce      ring RS + ring AG                              -> 2(g-1)*m
  all_gather      m = the FULL gathered size                     -> (g-1)*m
  reduce_scatter  m = the FULL input size                        -> (g-1)*m
Reductions add contributions in ascending group order, in fp64.
The ledger counts elements sent and received per (primitive, group, rank), and
sum(sent) == sum(received).
"""
from __future__ import annotations

from collections import defaultdict
from fractions import Fraction

import numpy as np


class Ledger:
    def __init__(self):
        self.sent = defaultdict(int)
        self.recv = defaultdict(int)

    def add(self, prim, group, src, dst, m):
        key_s = (prim, tuple(group), src)
        key_r = (prim, tuple(group), dst)
        self.sent[key_s] += m
        self.recv[key_r] += m

    def total(self, prim=None) -> int:
        return sum(v for (p, _, _), v in self.sent.items() if prim is None or p == prim)

    def total_received(self) -> int:
        return sum(self.recv.values())

    def per_rank_sent(self) -> dict:
        out = defaultdict(int)
        for (_, _, r), v in self.sent.items():
            out[r] += v
        return dict(out)


class Fabric:
    """Collectives over explicit per-rank buffers (dict rank -> ndarray)."""

    def __init__(self):
        self.ledger = Ledger()

    # -- each collective takes the group (ordered member list) and the per-rank inputs --
    def broadcast(self, group, root, payload):
        """Returns {member: copy of payload}."""
        if root not in group:
            raise ValueError("RootNotInGroup")
        m = np.asarray(payload).size
        out = {}
        for r in group:
            out[r] = np.array(payload, dtype=np.float64, copy=True)
            if r != root:
                self.ledger.add("broadcast", group, root, r, m)
        return out

    def reduce(self, group, root, parts: dict):
        """Sum of parts[r] over the group, ascending order, delivered to the root."""
        if root not in group:
            raise ValueError("RootNotInGroup")
        shapes = {np.shape(parts[r]) for r in group}
        if len(shapes) != 1:
            raise ValueError("ShapeMismatch")
        acc = np.zeros(next(iter(shapes)), dtype=np.float64)
        for r in group:
            acc = acc + np.asarray(parts[r], dtype=np.float64)
            if r != root:
                self.ledger.add("reduce", group, r, root, np.size(parts[r]))
        return acc

    def all_reduce(self, group, parts: dict):
        """Every member gets the ascending-order sum. Ledger: ring RS+AG."""
        shapes = {np.shape(parts[r]) for r in group}
        if len(shapes) != 1:
            raise ValueError("ShapeMismatch")
        g = len(group)
        acc = np.zeros(next(iter(shapes)), dtype=np.float64)
        for r in group:
            acc = acc + np.asarray(parts[r], dtype=np.float64)
        m = acc.size
        if g > 1:
            # ring: 2(g-1) steps, each member sends m/g elements per step
            for s in range(2 * (g - 1)):
                for idx, r in enumerate(group):
                    self.ledger.add("all_reduce", group, r, group[(idx + 1) % g], Fraction(m, g))
        return {r: acc.copy() for r in group}

    def all_gather(self, group, parts: dict, axis=0):
        """Concatenate the members' pieces in ascending group order."""
        pieces = [np.asarray(parts[r], dtype=np.float64) for r in group]
        full = np.concatenate(pieces, axis=axis)
        g = len(group)
        for idx, r in enumerate(group):
            for jdx, t in enumerate(group):
                if t != r:
                    self.ledger.add("all_gather", group, r, t, pieces[idx].size)
        return {r: full.copy() for r in group}

    def reduce_scatter(self, group, parts: dict, axis=0):
        """Member at position k gets the k-th of g equal slices of the ascending-order sum."""
        g = len(group)
        shapes = {np.shape(parts[r]) for r in group}
        if len(shapes) != 1:
            raise ValueError("ShapeMismatch")
        shape = next(iter(shapes))
        if shape[axis] % g:
            raise ValueError("IndivisibleLength")
        acc = np.zeros(shape, dtype=np.float64)
        for r in group:
            acc = acc + np.asarray(parts[r], dtype=np.float64)
        slices = np.split(acc, g, axis=axis)
        piece = acc.size // g
        for idx, r in enumerate(group):
            for jdx, t in enumerate(group):
                if t != r:
                    # r sends t its contribution to t's slice
                    self.ledger.add("reduce_scatter", group, r, t, piece)
        return {r: slices[idx].copy() for idx, r in enumerate(group)}
