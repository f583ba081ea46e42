"""Entries of full-size outputs computed one by one. TEST INFRASTRUCTURE ONLY.

For the BASELINE.json full sizes (e.g. M = K = N = 16384) the dense fp64 product is hours of
CPU work, but every entry of Y = alpha X.W + b, dX = alpha dY.W^T, dW = alpha X^T.dY and
db = 1^T dY is a single dot product of one row / column of the generator-defined inputs
(synth's counter-based generator gives any row or column directly). This module evaluates
those definitions (reading A1) entry by entry in fp64; the test pins it to the
dense oracle on small sizes.
"""
from __future__ import annotations

import numpy as np

import synth


def _rows(spec, tid, R, C, idx):
    return synth.rows_of(spec["seed"], tid, R, C, idx, spec["kind"], spec.get("scale_" + str(tid), 1.0),
                         spec["dtype"]).astype(np.float64)


def _cols(spec, tid, R, C, idx):
    return synth.cols_of(spec["seed"], tid, R, C, idx, spec["kind"], spec.get("scale_" + str(tid), 1.0),
                         spec["dtype"]).astype(np.float64)


def layer_spec(seed, M, K, N, layer=0, kind="uniform", dtype="bf16"):
    """The generator recipe of synth.layer_inputs (X, W Xavier, dY, bias) for one layer."""
    tx, tw = synth.layer_tid(layer, synth.TID_X), synth.layer_tid(layer, synth.TID_W)
    tdy, tb = synth.layer_tid(layer, synth.TID_DY), synth.layer_tid(layer, synth.TID_BIAS)
    spec = {"seed": seed, "M": M, "K": K, "N": N, "kind": kind, "dtype": dtype,
            "tx": tx, "tw": tw, "tdy": tdy, "tb": tb}
    spec["scale_" + str(tw)] = synth.xavier_scale(K, N) if kind == "uniform" else 1.0
    return spec


def y_entries(spec, rows, cols, alpha=1.0, with_bias=False):
    """Y[r, c] = alpha * sum_k X[r,k] W[k,c] (+ b[c])."""
    M, K, N = spec["M"], spec["K"], spec["N"]
    Xr = _rows(spec, spec["tx"], M, K, rows)          # [n, K]
    Wc = _cols(spec, spec["tw"], K, N, cols)          # [K, n]
    out = alpha * np.einsum("ik,ki->i", Xr, Wc)
    if with_bias:
        out = out + _rows(spec, spec["tb"], 1, N, np.zeros(len(cols), dtype=np.int64))[
            np.arange(len(cols)), np.asarray(cols)]
    return out


def dx_entries(spec, rows, ks, alpha=1.0):
    """dX[r, k] = alpha * sum_n dY[r,n] W[k,n]."""
    M, K, N = spec["M"], spec["K"], spec["N"]
    dYr = _rows(spec, spec["tdy"], M, N, rows)
    Wr = _rows(spec, spec["tw"], K, N, ks)
    return alpha * np.einsum("in,in->i", dYr, Wr)


def dw_entries(spec, ks, cols, alpha=1.0):
    """dW[k, c] = alpha * sum_m X[m,k] dY[m,c]."""
    M, K, N = spec["M"], spec["K"], spec["N"]
    Xc = _cols(spec, spec["tx"], M, K, ks)
    dYc = _cols(spec, spec["tdy"], M, N, cols)
    return alpha * np.einsum("mi,mi->i", Xc, dYc)


def db_entries(spec, cols):
    """db[c] = sum_m dY[m,c]."""
    M, N = spec["M"], spec["N"]
    return _cols(spec, spec["tdy"], M, N, cols).sum(axis=0)


def sample_indices(seed, n, *bounds):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, b, size=n) for b in bounds]


def stratified_indices(seed, extent, block=128):
    """One index inside every `block`-wide slab of [0, extent) (random offset per slab, the last
    slab may be ragged). Crossing a row sample with a column sample from this puts one checked
    entry in every block x block output tile, so a single wrong GEMM tile cannot go unseen."""
    rng = np.random.default_rng(seed)
    lo = np.arange(0, extent, block, dtype=np.int64)
    width = np.minimum(block, extent - lo)
    return lo + rng.integers(0, width)


# ---------------------------------------------------------------- row x column grids, one layer

def y_grid(spec, rows, cols, alpha=1.0):
    """Y[rows][:, cols] = alpha * X[rows, :] . W[:, cols] (every (row, col) pair)."""
    M, K, N = spec["M"], spec["K"], spec["N"]
    return alpha * (_rows(spec, spec["tx"], M, K, rows) @ _cols(spec, spec["tw"], K, N, cols))


def dx_grid(spec, rows, ks, alpha=1.0):
    """dX[rows][:, ks] = alpha * dY[rows, :] . W[ks, :]^T."""
    M, K, N = spec["M"], spec["K"], spec["N"]
    return alpha * (_rows(spec, spec["tdy"], M, N, rows) @ _rows(spec, spec["tw"], K, N, ks).T)


def dw_grid(spec, ks, cols, alpha=1.0):
    """dW[ks][:, cols] = alpha * X[:, ks]^T . dY[:, cols]."""
    M, K, N = spec["M"], spec["K"], spec["N"]
    return alpha * (_cols(spec, spec["tx"], M, K, ks).T @ _cols(spec, spec["tdy"], M, N, cols))


# ---------------------------------------------------------------- the two-layer chain

def _mm(A, B, chunk=2048):
    """fp64 A . B with A converted to fp64 one block of rows at a time (memory only: each output
    entry is still one full-length dot product)."""
    B = np.asarray(B, np.float64)
    out = np.empty((A.shape[0], B.shape[1]), dtype=np.float64)
    for r in range(0, A.shape[0], chunk):
        out[r:r + chunk] = np.asarray(A[r:r + chunk], np.float64) @ B
    return out


def chain2_grids(X, W1, W2, dY, idx):
    """Sampled outputs of the paper's range-test model, two linear layers ("a model
    which consists of two linear layers"; reading A14; activations ignored), from the
    global inputs X [M,K], W1 [K,H], W2 [H,N], dY (= dY2) [M,N]:

        Y1 = X.W1,  Y2 = Y1.W2;   dY1 = dY.W2^T,  dW2 = Y1^T.dY,  dX = dY1.W1^T,  dW1 = X^T.dY1

    idx maps each output to its (row sample, column sample):
        "Y": rows of M, cols of N;  "dX": rows of M, cols of K;
        "dW1": rows of K, cols of H;  "dW2": rows of H, cols of N.
    Returns {name: fp64 [len(rows), len(cols)]}. Only the rows / columns of Y1 and dY1 the
    samples touch are formed (a row of Y1 needs all of W1, a column of Y1 all of X)."""
    out = {}
    if "Y" in idx:
        r, c = idx["Y"]
        Y1r = _mm(X[r], W1)                                  # Y1[r, :]
        out["Y"] = Y1r @ np.asarray(W2[:, c], np.float64)
    if "dX" in idx:
        r, c = idx["dX"]
        dY1r = _mm(dY[r], np.asarray(W2, np.float64).T)      # dY1[r, :]
        out["dX"] = dY1r @ np.asarray(W1[c, :], np.float64).T
    if "dW1" in idx:
        r, c = idx["dW1"]
        dY1c = _mm(dY, np.asarray(W2[c, :], np.float64).T)   # dY1[:, c]
        out["dW1"] = np.asarray(X[:, r], np.float64).T @ dY1c
    if "dW2" in idx:
        r, c = idx["dW2"]
        Y1c = _mm(X, np.asarray(W1[:, r], np.float64))       # Y1[:, r]
        out["dW2"] = Y1c.T @ np.asarray(dY[:, c], np.float64)
    return out
