"""GeLU between the linears of a Transformer MLP, in the tensor-parallel layouts.
TEST INFRASTRUCTURE ONLY (imported by tests/ only).

SURVEY 8(f) NEXT-2: "bias+GeLU epilogue". The paper ignores activations for its range tests
 but its models (ViT, GPT, BERT) put GeLU after the first MLP linear.
Definition (Hendrycks & Gimpel, the exact erf form used by ViT and BERT; reading N2):

    gelu(z)  = z * Phi(z) = 0.5 z (1 + erf(z / sqrt 2))
    gelu'(z) = Phi(z) + z * phi(z),   phi(z) = exp(-z^2 / 2) / sqrt(2 pi)

A layer with activation computes Z = alpha X.W + b (the linear layer of programs.py, any
mode), then Y = gelu(Z) elementwise on each rank's Y shard; backward takes dL/dY, forms
dZ = dY * gelu'(Z) on the same shard and runs the linear layer's backward with dZ (db = 1^T dZ).
Elementwise on the Y layout, so no communication is added in any mode.
"""
from __future__ import annotations

import math

import numpy as np

from . import programs


def _erf(z):
    return np.vectorize(math.erf, otypes=[np.float64])(np.asarray(z, np.float64))


def gelu(z):
    z = np.asarray(z, np.float64)
    return 0.5 * z * (1.0 + _erf(z / math.sqrt(2.0)))


def gelu_grad(z):
    z = np.asarray(z, np.float64)
    Phi = 0.5 * (1.0 + _erf(z / math.sqrt(2.0)))
    phi = np.exp(-0.5 * z * z) / math.sqrt(2.0 * math.pi)
    return Phi + z * phi


def act_layer_fwd(grid, spec, Xs, Ws, bs=None, alpha=1.0, fab=None):
    """Per-rank (Y = gelu(Z) shards, saved) with saved = (linear saved, Z shards)."""
    Zs, sv = programs.layer_fwd(grid, spec, Xs, Ws, bs, alpha, fab)
    return {r: gelu(z) for r, z in Zs.items()}, (sv, Zs)


def act_layer_bwd(grid, spec, dYs, Xs, Ws, alpha, fab, saved):
    """(dX, dW, db) shards of Y = gelu(alpha X.W + b) given dL/dY shards."""
    sv, Zs = saved
    dZs = {r: np.asarray(dYs[r], np.float64) * gelu_grad(Zs[r]) for r in dYs}
    return programs.layer_bwd(grid, spec, dZs, Xs, Ws, alpha, fab, sv)
