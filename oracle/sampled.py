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
