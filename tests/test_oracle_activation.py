"""Pins of the GeLU oracle (oracle/activation.py) to things other than itself: PyTorch's fp64
gelu (library routine, exact erf form) and its autograd, the identity gelu(z) - gelu(-z) = z,
limits, finite differences, and the rank-by-rank activation layer == dense on every mode."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import activation as act
from oracle import dense
from oracle.fabric import Fabric
from oracle.grid import build_grid
from oracle.shards import LayerSpec, gather_full, shard


def test_matches_torch_fp64():
    z = np.linspace(-8, 8, 1001)
    t = torch.tensor(z, requires_grad=True)
    y = torch.nn.functional.gelu(t, approximate="none")
    assert np.allclose(act.gelu(z), y.detach().numpy(), rtol=0, atol=1e-15)
    y.sum().backward()
    assert np.allclose(act.gelu_grad(z), t.grad.numpy(), rtol=0, atol=1e-14)


def test_identities_and_limits():
    z = np.linspace(-5, 5, 101)
    assert np.allclose(act.gelu(z) - act.gelu(-z), z, atol=1e-14)   # z Phi(z) + z Phi(-z) = z
    assert act.gelu(0.0) == 0.0 and act.gelu_grad(0.0) == 0.5
    assert abs(act.gelu(40.0) - 40.0) < 1e-12 and abs(act.gelu(-40.0)) < 1e-12
    assert abs(float(act.gelu(1.0)) - 0.5 * (1 + math.erf(1 / math.sqrt(2)))) < 1e-15


def test_gradient_finite_differences():
    z = np.array([-3.0, -1.0, -0.1, 0.0, 0.3, 1.7, 4.0])
    h = 1e-6
    fd = (act.gelu(z + h) - act.gelu(z - h)) / (2 * h)
    assert np.allclose(act.gelu_grad(z), fd, atol=1e-8)


GRIDS = [("1d", 4, 1, "col", 0), ("1d", 4, 1, "row", 0), ("2d", 4, 1, "col", 0),
         ("2.5d", 8, 2, "col", 0), ("3d", 8, 1, "col", 0), ("3d", 8, 1, "col", 1)]


@pytest.mark.parametrize("g", GRIDS, ids=lambda g: "-".join(map(str, g)))
def test_rank_programs_equal_dense(g):
    mode, p, d, split, par = g
    M, K, N = 32, 16, 24
    grid = build_grid(mode, p, d)
    spec = LayerSpec(M, K, N, split_1d=split, parity=par)
    X, W, dY, b = synth.layer_inputs(4, M, K, N, with_bias=True)
    Z = dense.linear_fwd(X, W, b, alpha=0.5)
    Yd = act.gelu(Z)
    dZ = dY * act.gelu_grad(Z)
    dXd, dWd, dbd = dense.linear_bwd(dZ, X, W, alpha=0.5)
    fab = Fabric()
    Xs, Ws = shard(grid, spec, X, "X"), shard(grid, spec, W, "W")
    Ys, sv = act.act_layer_fwd(grid, spec, Xs, Ws, shard(grid, spec, b, "B"), 0.5, fab)
    assert np.allclose(gather_full(grid, spec, Ys, "Y"), Yd, atol=1e-12)
    dXs, dWs, dbs = act.act_layer_bwd(grid, spec, shard(grid, spec, dY, "Y"), Xs, Ws, 0.5, fab, sv)
    assert np.allclose(gather_full(grid, spec, dXs, "X"), dXd, atol=1e-12)
    assert np.allclose(gather_full(grid, spec, dWs, "W"), dWd, atol=1e-12)
    assert np.allclose(gather_full(grid, spec, dbs, "B"), dbd, atol=1e-12)
