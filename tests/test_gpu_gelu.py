"""GPU parity of the GeLU activation layer (TP_FLAG_GELU): Y = gelu(alpha
X.W + b) forward and dL/dY -> (dX, dW, db) backward on every TP mode, against the oracle
(oracle/activation.py, pinned in tests/test_oracle_activation.py). In-process ranks on cuda:0."""
import numpy as np
import pytest
import torch

import synth
from oracle import activation as act
from oracle import dense

from tp_harness import gather, rel_fro, spec_of, tp_layer

pytestmark = pytest.mark.gpu

GELU, FUSED = 0x8, 0x4
GRIDS = [("1d", 1, 1, 0, 0), ("1d", 4, 1, 0, 0), ("1d", 4, 1, 1, 0), ("2d", 4, 1, 0, 0),
         ("2.5d", 8, 2, 0, 0), ("3d", 8, 1, 0, 0), ("3d", 8, 1, 0, 1)]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def _dense(X, W, b, dY, alpha):
    Z = dense.linear_fwd(X, W, b, alpha=alpha)
    dX, dW, db = dense.linear_bwd(dY * act.gelu_grad(Z), X, W, alpha=alpha)
    return act.gelu(Z), dX, dW, db


@pytest.mark.parametrize("grid", GRIDS, ids=lambda g: "-".join(map(str, g)))
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_gelu_layer_vs_oracle(api, grid, dtype):
    mode, p, d, split, par = grid
    M, K, N = (520, 384, 640) if dtype == "bf16" else (48, 64, 64)
    X, W, dY, b = synth.layer_inputs(13, M, K, N, dtype=dtype, with_bias=True)
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, dtype, split, par, GELU, alpha=0.75)
    Yr, dXr, dWr, dbr = _dense(X, W, b, dY, 0.75)
    spec = spec_of(M, K, N, split, par)
    tol = 1e-2 if dtype == "bf16" else 1e-5
    assert rel_fro(gather(mode, p, d, spec, per, "Y", "Y"), Yr) <= tol
    assert rel_fro(gather(mode, p, d, spec, per, "dX", "X"), dXr) <= tol
    assert rel_fro(gather(mode, p, d, spec, per, "dW", "W"), dWr) <= tol
    assert rel_fro(gather(mode, p, d, spec, per, "dB", "B"), dbr) <= tol


@pytest.mark.parametrize("mode,p,d,par", [("2d", 4, 1, 0), ("3d", 8, 1, 1)])
def test_gelu_with_fused_forward(api, mode, p, d, par):
    """GeLU on top of the fused peer-panel forward; the backward's dZ is a library temporary
    (not a registered buffer), so the backward takes the collective schedule."""
    M, K, N = 544, 576, 400
    X, W, dY, b = synth.layer_inputs(17, M, K, N, with_bias=True)
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, "bf16", 0, par, GELU | FUSED)
    Yr, dXr, dWr, dbr = _dense(X, W, b, dY, 1.0)
    spec = spec_of(M, K, N, 0, par)
    for key, t, ref in (("Y", "Y", Yr), ("dX", "X", dXr), ("dW", "W", dWr), ("dB", "B", dbr)):
        assert rel_fro(gather(mode, p, d, spec, per, key, t), ref) <= 1e-2, key
