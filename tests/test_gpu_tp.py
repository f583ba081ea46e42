"""Multi-rank parity of every TP mode on ONE B200: the C ABI's schedules run with the
in-process transport (one host thread per rank on cuda:0) and are compared element by
element with the oracle's rank-by-rank fp64 program (SURVEY 8(a) a-3 .. a-10).

Grids covered: every grid SURVEY 8(a)-1 lists at 1/2/4/8 GPUs (1D p in {1,2,4,8} col and
row; 2D q in {1,2}; 2.5D (d=1,q=2)@4, (d=2,q=2)@8 with both weight layouts; 3D l in {1,2}
both parities), plus 2D q=3 (a ragged, non-power-of-two grid).
"""
import numpy as np
import pytest
import torch

import synth
from oracle import dense, programs
from oracle.grid import build_grid

from tp_harness import gather, oracle_layer, rel_fro, spec_of, tp_layer

pytestmark = pytest.mark.gpu

GRIDS = [
    ("1d", 1, 1, dict(split_1d=0)), ("1d", 2, 1, dict(split_1d=0)), ("1d", 4, 1, dict(split_1d=0)),
    ("1d", 8, 1, dict(split_1d=0)), ("1d", 2, 1, dict(split_1d=1)), ("1d", 8, 1, dict(split_1d=1)),
    ("2d", 1, 1, {}), ("2d", 4, 1, {}), ("2d", 9, 1, {}),
    ("2.5d", 4, 1, {}), ("2.5d", 8, 2, {}), ("2.5d", 8, 2, dict(flags=1)),
    ("3d", 1, 1, {}), ("3d", 8, 1, dict(parity=0)), ("3d", 8, 1, dict(parity=1)),
]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def _ids(g):
    m, p, d, kw = g
    return f"{m}-p{p}-d{d}-" + "-".join(f"{k}{v}" for k, v in kw.items())


def _shapes(mode, p, d):
    """Global shapes spanning several 128-row tiles with ragged tails, TMA-legal strides."""
    if mode == "2d" and p == 9:
        return 390, 264, 408           # shards 130 x 88 x 136
    return 520, 384, 640               # 2D: 260x192x320; 3D: 130 rows, K/l 192, N/l 320


@pytest.mark.parametrize("grid", GRIDS, ids=_ids)
@pytest.mark.parametrize("with_bias", [False, True])
def test_layer_bf16_vs_oracle(api, grid, with_bias):
    mode, p, d, kw = grid
    M, K, N = _shapes(mode, p, d)
    X, W, dY, b = synth.layer_inputs(42, M, K, N, with_bias=True)
    b = b if with_bias else None
    split = kw.get("split_1d", 0)
    parity = kw.get("parity", 0)
    flags = kw.get("flags", 0)
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, "bf16", split, parity, flags, alpha=0.5)
    spec = spec_of(M, K, N, split, parity, flags)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY, b, alpha=0.5)
    assert rel_fro(gather(mode, p, d, spec, per, "Y", "Y"), Yr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dX", "X"), dXr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dW", "W"), dWr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dB", "B"), dbr) <= 1e-2


@pytest.mark.parametrize("grid", GRIDS, ids=_ids)
def test_layer_exact_integer_bit_equal(api, grid):
    """Ternary inputs with M, K, N <= 256: every partial, every collective sum and every
    output is an exact small integer, so the GPU must be bit-equal to the oracle (A17)."""
    mode, p, d, kw = grid
    M, K, N = (144, 256, 192) if not (mode == "2d" and p == 9) else (144, 216, 216)
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    split, parity, flags = kw.get("split_1d", 0), kw.get("parity", 0), kw.get("flags", 0)
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, None, "bf16", split, parity, flags)
    spec = spec_of(M, K, N, split, parity, flags)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY)
    assert np.array_equal(gather(mode, p, d, spec, per, "Y", "Y"), Yr)
    assert np.array_equal(gather(mode, p, d, spec, per, "dX", "X"), dXr)
    assert np.array_equal(gather(mode, p, d, spec, per, "dW", "W"), dWr)
    assert np.array_equal(gather(mode, p, d, spec, per, "dB", "B"), dbr)


@pytest.mark.parametrize("mode,p,d", [("2d", 4, 1), ("1d", 4, 1), ("2.5d", 8, 2), ("3d", 8, 1)])
def test_config_c1_fp32(api, mode, p, d):
    """BASELINE configs[0]: batch 16 x hidden 64, fp32 (SIMT path), 1e-5 bar."""
    M, H = 16, 64
    X, W, dY, b = synth.layer_inputs(42, M, H, H, dtype="fp32", with_bias=True)
    per = tp_layer(api, mode, p, d, M, H, H, X, W, dY, b, "fp32")
    spec = spec_of(M, H, H)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY, b)
    for key, t, ref in (("Y", "Y", Yr), ("dX", "X", dXr), ("dW", "W", dWr), ("dB", "B", dbr)):
        assert rel_fro(gather(mode, p, d, spec, per, key, t), ref) <= 1e-5


def test_skip_dx(api):
    M, K, N = 520, 384, 640
    X, W, dY, _ = synth.layer_inputs(1, M, K, N)
    per = tp_layer(api, "2d", 4, 1, M, K, N, X, W, dY, want_dx=False)
    spec = spec_of(M, K, N)
    _, _, dWr, _ = oracle_layer("2d", 4, 1, spec, X, W, dY)
    assert rel_fro(gather("2d", 4, 1, spec, per, "dW", "W"), dWr) <= 1e-2


def test_degenerate_zero_batch(api):
    """M = 0: Y and dX are empty, dW = X^T dY = 0 and db = 0 must still be written."""
    K, N = 64, 128
    X, W, dY = (np.zeros((0, K), np.float32), synth.tensor(1, 1, K, N), np.zeros((0, N), np.float32))
    per = tp_layer(api, "2d", 4, 1, 0, K, N, X, W, dY)
    for r in range(4):
        assert not per[r]["dW"].any() and not per[r]["dB"].any()
