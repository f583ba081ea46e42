"""Dense fp64 linear layer: the plain definition every TP mode reaches exactly.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:L391 "computing a matrix multiplication Y=WX where X is of shape (b,s,h), W is
of shape (h,h)" - read (reading A1) as Y = X.W with X flattened to
[M = b*s, K] row-major and W [K, N] (input-major), because only this convention
makes the Megatron column/row split of P:L488 well-typed. The backward is the
chain rule of that product ("derivation is standard"):
    dX = alpha * dY . W^T,  dW = alpha * X^T . dY,  db = 1^T . dY.
Bias is not in the paper (reading A16); it is optional here.
Activations between the two linears are ignored ("The activation
functions and normalization layers are ignored").
"""
from __future__ import annotations

import numpy as np


def f64(a):
    return np.asarray(a, dtype=np.float64)


def matmul(A, B):
    """fp64 matrix product (library primitive)."""
    A, B = f64(A), f64(B)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise ValueError(f"ShapeMismatch {A.shape} x {B.shape}")
    return A @ B


def linear_fwd(X, W, b=None, alpha=1.0):
    """Y = alpha * X.W (+ b broadcast over rows)."""
    Y = alpha * matmul(X, W)
    if b is not None:
        Y = Y + f64(b)[None, :]
    return Y


def linear_bwd(dY, X, W, alpha=1.0):
    """(dX, dW, db) of Y = alpha*X.W + b."""
    dY = f64(dY)
    dX = alpha * matmul(dY, f64(W).T)
    dW = alpha * matmul(f64(X).T, dY)
    db = dY.sum(axis=0)
    return dX, dW, db


def mlp2_fwd(X, W1, W2, alpha=1.0):
    """Two linear layers (the paper's range-test model): Y1 = X.W1, Y2 = Y1.W2."""
    Y1 = linear_fwd(X, W1, alpha=alpha)
    Y2 = linear_fwd(Y1, W2, alpha=alpha)
    return Y1, Y2


def mlp2_bwd(dY2, X, Y1, W1, W2, alpha=1.0):
    """dY1 = dY2.W2^T, dW2 = Y1^T.dY2, dX = dY1.W1^T, dW1 = X^T.dY1."""
    dY1, dW2, _ = linear_bwd(dY2, Y1, W2, alpha)
    dX, dW1, _ = linear_bwd(dY1, X, W1, alpha)
    return dX, dW1, dW2, dY1
