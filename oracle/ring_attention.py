"""Ring Self-Attention forward (sequence parallelism). TEST INFRASTRUCTURE ONLY.

SURVEY 8(f) NEXT-3; PAPER P:L596-615 (Sequence Parallelism):
  "the input data is split along the sequence dimension and each device only keeps the
   sub-sequence" ... "Attention(Q, K, V) = softmax(QK^T / sqrt(d_k)) V" ... "the key
   embedding is first multiplied with the query embedding on the local device, and then
   transferred to the next device for N-1 times ... In this way, the partial attention score
   with respect to the local sub-sequence can be obtained. The final attention output AV can
   be calculated in a similar fashion."
SPEC S:L361-414 (ring_attention) fixes the realisation this oracle follows: equal-size
contiguous shards in rank order; pass 1 circulates K blocks (N-1 ring shifts), placing the
score block of K's originating rank in its columns; softmax row-wise over the assembled
local rows (two-pass, reading N3); pass 2 circulates V blocks and accumulates A[:, blk] V_blk.
Single head per call; heads are independent (batch them by looping).

Ledger: each ring shift moves every rank's (s/N) x d block to its successor -- per pass
(N-1) * N * (s/N) * d = (N-1) s d elements; K pass + V pass = 2 (N-1) s d (S:L377 volume law).
"""
from __future__ import annotations

import math

import numpy as np

from .fabric import Ledger


class IndivisibleSequence(ValueError):
    """s is not divisible by the ring size."""


def attention(Q, K, V, scale=None):
    """Dense softmax(Q K^T * scale) V in fp64 (scale defaults to 1/sqrt(d_k))."""
    Q, K, V = (np.asarray(a, np.float64) for a in (Q, K, V))
    scale = 1.0 / math.sqrt(Q.shape[1]) if scale is None else scale
    S = (Q @ K.T) * scale
    S = S - S.max(axis=1, keepdims=True)
    A = np.exp(S)
    A = A / A.sum(axis=1, keepdims=True)
    return A @ V, A


def shards(X, N):
    s = X.shape[0]
    if s % N:
        raise IndivisibleSequence(f"s={s} not divisible by N={N}")
    b = s // N
    return {r: np.asarray(X[r * b:(r + 1) * b], np.float64) for r in range(N)}


def ring_attention(Qs: dict, Ks: dict, Vs: dict, scale=None, ledger: Ledger | None = None):
    """Rank-by-rank RSA forward. Returns ({rank: output rows}, {rank: assembled scores})."""
    N = len(Qs)
    b, d = np.shape(Qs[0])
    s = b * N
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    group = tuple(range(N))
    # pass 1: K ring. At step t rank r holds the K block that originated on rank (r - t) mod N.
    held = {r: np.asarray(Ks[r], np.float64) for r in range(N)}
    S = {r: np.zeros((b, s)) for r in range(N)}
    for t in range(N):
        for r in range(N):
            j = (r - t) % N
            S[r][:, j * b:(j + 1) * b] = (np.asarray(Qs[r], np.float64) @ held[r].T) * scale
        if t < N - 1:  # ring shift: r sends to r+1
            if ledger is not None:
                for r in range(N):
                    ledger.add("ring_k", group, r, (r + 1) % N, b * d)
            held = {r: held[(r - 1) % N] for r in range(N)}
    # row-wise softmax over the assembled local rows (max-subtracted, two passes)
    A = {}
    for r in range(N):
        e = np.exp(S[r] - S[r].max(axis=1, keepdims=True))
        A[r] = e / e.sum(axis=1, keepdims=True)
    # pass 2: V ring; accumulate A[:, block j] . V_j
    held = {r: np.asarray(Vs[r], np.float64) for r in range(N)}
    O = {r: np.zeros((b, np.shape(Vs[0])[1])) for r in range(N)}
    for t in range(N):
        for r in range(N):
            j = (r - t) % N
            O[r] = O[r] + A[r][:, j * b:(j + 1) * b] @ held[r]
        if t < N - 1:
            if ledger is not None:
                for r in range(N):
                    ledger.add("ring_v", group, r, (r + 1) % N, b * np.shape(Vs[0])[1])
            held = {r: held[(r - 1) % N] for r in range(N)}
    return O, S


# ------------------------------------------------------------------------------- backward
# The paper describes the forward only; the backward is the chain rule of the same definition
# (reading N4), organised on the same ring:
#   P = softmax(S), S = scale Q K^T, O = P V
#   dV = P^T dO,  dP = dO V^T,  dS = P * (dP - rowsum(P * dP)),  dQ = scale dS K,
#   dK = scale dS^T Q.
# Rank r holds query rows r; it recomputes its score rows with the K ring (as the forward),
# forms dP over the V ring, dQ over the K ring, and its contributions P_r[:, j]^T dO_r and
# scale dS_r[:, j]^T Q_r to every key block j, which a reduce-scatter over the ring sums into
# the owner of block j.


def attention_bwd(Q, K, V, dO, scale=None):
    """Dense gradients (dQ, dK, dV) of O = softmax(Q K^T scale) V, fp64."""
    Q, K, V, dO = (np.asarray(a, np.float64) for a in (Q, K, V, dO))
    scale = 1.0 / math.sqrt(Q.shape[1]) if scale is None else scale
    _, P = attention(Q, K, V, scale)
    dV = P.T @ dO
    dP = dO @ V.T
    dS = P * (dP - (P * dP).sum(axis=1, keepdims=True))
    return scale * dS @ K, scale * dS.T @ Q, dV


def ring_attention_bwd(Qs: dict, Ks: dict, Vs: dict, dOs: dict, scale=None,
                       ledger: Ledger | None = None):
    """Rank-by-rank RSA backward: ({r: dQ_r}, {r: dK_r}, {r: dV_r})."""
    N = len(Qs)
    b, d = np.shape(Qs[0])
    s = b * N
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    group = tuple(range(N))
    _, S = ring_attention(Qs, Ks, Vs, scale, ledger)    # K ring (recompute) + V ring
    P = {}
    for r in range(N):
        e = np.exp(S[r] - S[r].max(axis=1, keepdims=True))
        P[r] = e / e.sum(axis=1, keepdims=True)
    # dP rows over the V ring
    held = {r: np.asarray(Vs[r], np.float64) for r in range(N)}
    dP = {r: np.zeros((b, s)) for r in range(N)}
    for t in range(N):
        for r in range(N):
            j = (r - t) % N
            dP[r][:, j * b:(j + 1) * b] = np.asarray(dOs[r], np.float64) @ held[r].T
        if t < N - 1:
            if ledger is not None:
                for r in range(N):
                    ledger.add("ring_v", group, r, (r + 1) % N, b * d)
            held = {r: held[(r - 1) % N] for r in range(N)}
    dS = {r: P[r] * (dP[r] - (P[r] * dP[r]).sum(axis=1, keepdims=True)) for r in range(N)}
    # dQ over the K ring
    held = {r: np.asarray(Ks[r], np.float64) for r in range(N)}
    dQ = {r: np.zeros((b, d)) for r in range(N)}
    for t in range(N):
        for r in range(N):
            j = (r - t) % N
            dQ[r] = dQ[r] + scale * dS[r][:, j * b:(j + 1) * b] @ held[r]
        if t < N - 1:
            if ledger is not None:
                for r in range(N):
                    ledger.add("ring_k", group, r, (r + 1) % N, b * d)
            held = {r: held[(r - 1) % N] for r in range(N)}
    # dK, dV: every rank's contribution to every key block, summed at the block's owner
    dK = {j: sum(scale * dS[r][:, j * b:(j + 1) * b].T @ np.asarray(Qs[r], np.float64)
                 for r in range(N)) for j in range(N)}
    dV = {j: sum(P[r][:, j * b:(j + 1) * b].T @ np.asarray(dOs[r], np.float64)
                 for r in range(N)) for j in range(N)}
    if ledger is not None and N > 1:  # two reduce-scatters of N blocks of b x d
        for r in range(N):
            ledger.add("reduce_scatter", group, r, r, 2 * (N - 1) * b * d)
    return dQ, dK, dV
