"""GPU parity of the Solomonik-style 2.5D layer (TP_FLAG_SOLOMONIK, reading
N5) against oracle/solomonik.py (pinned in tests/test_oracle_solomonik.py): every layer holds
the 2D block layout, layer dep runs its 1/d of the SUMMA steps, Y is all-reduced and dX / dW
depth-broadcast. In-process ranks on cuda:0 (LOCAL transport)."""
import numpy as np
import pytest
import torch

import synth
from oracle import solomonik as so
from oracle.fabric import Fabric
from oracle.grid import build_grid
from oracle.shards import LayerSpec

from tp_harness import rel_fro, tp_layer

pytestmark = pytest.mark.gpu

SOLOMONIK = 0x20


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def oracle(p, d, M, K, N, X, W, dY, b, alpha):
    grid, spec = build_grid("2.5d", p, d), LayerSpec(M, K, N)
    Xs, Ws = so.shard(grid, spec, X, "X"), so.shard(grid, spec, W, "W")
    bs = so.shard(grid, spec, b, "B") if b is not None else None
    fab = Fabric()
    Y = so.fwd(grid, Xs, Ws, bs, alpha, fab)
    dX, dW, db = so.bwd(grid, so.shard(grid, spec, dY, "Y"), Xs, Ws, alpha, fab)
    g = lambda sh, t: so.gather_full(grid, spec, sh, t)
    return grid, spec, g(Y, "Y"), g(dX, "X"), g(dW, "W"), g(db, "B")


@pytest.mark.parametrize("p,d,M,K,N", [
    (8, 2, 520, 400, 656),     # q=2, d=2: one step per layer, ragged GEMM tiles
    (4, 1, 264, 144, 208),     # q=2, d=1: plain SUMMA
    (32, 2, 512, 384, 640),    # q=4, d=2: two steps per layer (double-buffered panels)
], ids=["q2d2", "q2d1", "q4d2"])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_solomonik_vs_oracle(api, p, d, M, K, N, dtype):
    X, W, dY, b = synth.layer_inputs(41, M, K, N, dtype=dtype, with_bias=True)
    per = tp_layer(api, "2.5d", p, d, M, K, N, X, W, dY, b, dtype, flags=SOLOMONIK, alpha=0.5)
    grid, spec, Yr, dXr, dWr, dbr = oracle(p, d, M, K, N, X, W, dY, b, 0.5)
    tol = 1e-2 if dtype == "bf16" else 1e-5
    # gather_full also checks that every layer's replica is bit-identical
    g = lambda key, t: so.gather_full(grid, spec, {r: per[r][key] for r in range(p)}, t)
    assert rel_fro(g("Y", "Y"), Yr) <= tol
    assert rel_fro(g("dX", "X"), dXr) <= tol
    assert rel_fro(g("dW", "W"), dWr) <= tol
    assert rel_fro(g("dB", "B"), dbr) <= tol


def test_solomonik_exact_integer(api):
    p, d, M, K, N = 8, 2, 272, 256, 272
    X, W, dY, _ = synth.layer_inputs(8, M, K, N, kind="ternary")
    per = tp_layer(api, "2.5d", p, d, M, K, N, X, W, dY, None, "bf16", flags=SOLOMONIK)
    grid, spec, Yr, dXr, dWr, _ = oracle(p, d, M, K, N, X, W, dY, None, 1.0)
    g = lambda key, t: so.gather_full(grid, spec, {r: per[r][key] for r in range(p)}, t)
    assert np.array_equal(g("Y", "Y"), Yr)
    assert np.array_equal(g("dX", "X"), dXr)
    assert np.array_equal(g("dW", "W"), dWr)


def test_solomonik_rejects_bad_grids(api):
    g = api.tp_grid_init("2.5d", 16, 0, 0, 4, 0, api.TP_TRANSPORT_NONE)  # q = 2, d = 4
    try:
        with pytest.raises(api.TPError):
            api.tp_shard_extent(g, api.desc(64, 64, 64, "bf16", flags=SOLOMONIK), "X")
    finally:
        api.tp_grid_destroy(g)
    g = api.tp_grid_init("2.5d", 8, 0, 0, 2, 0, api.TP_TRANSPORT_NONE)
    try:
        with pytest.raises(api.TPError):  # excludes the depth-sharded weight layout
            api.tp_shard_extent(g, api.desc(64, 64, 64, "bf16", flags=SOLOMONIK | 0x1), "X")
    finally:
        api.tp_grid_destroy(g)
