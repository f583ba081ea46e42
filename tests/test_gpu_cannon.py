"""GPU parity of Cannon's 2D forward (TP_FLAG_CANNON) against the oracle's
Cannon and SUMMA programs (oracle/cannon.py, pinned in tests/test_oracle_cannon.py) on 2D
q = 2, 3, 4 and 2.5D planes (d = 2, both weight layouts); in-process ranks on cuda:0."""
import numpy as np
import pytest
import torch

import synth
from oracle import cannon
from oracle.fabric import Fabric
from oracle.grid import build_grid
from oracle.shards import gather_full, shard

from tp_harness import gather, oracle_layer, rel_fro, spec_of, tp_layer

pytestmark = pytest.mark.gpu
CANNON = 0x10


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


@pytest.mark.parametrize("mode,p,d,flags", [("2d", 4, 1, 0), ("2d", 9, 1, 0), ("2d", 16, 1, 0),
                                            ("2.5d", 8, 2, 0), ("2.5d", 8, 2, 1)])
def test_cannon_vs_oracle(api, mode, p, d, flags):
    q = {4: 2, 9: 3, 16: 4, 8: 2}[p]
    M, K, N = 48 * q * d, 40 * q * d, 56 * q
    X, W, dY, b = synth.layer_inputs(21, M, K, N, with_bias=True)
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, "bf16", 0, 0, CANNON | flags, alpha=0.5)
    spec = spec_of(M, K, N, 0, 0, flags)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY, b, alpha=0.5)
    assert rel_fro(gather(mode, p, d, spec, per, "Y", "Y"), Yr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dX", "X"), dXr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dW", "W"), dWr) <= 1e-2
    if mode == "2d":  # the oracle's Cannon program itself
        grid = build_grid("2d", p)
        Yc = cannon.cannon_fwd(grid, shard(grid, spec, X, "X"), shard(grid, spec, W, "W"),
                               shard(grid, spec, b, "B"), 0.5, Fabric())
        assert rel_fro(gather(mode, p, d, spec, per, "Y", "Y"), gather_full(grid, spec, Yc, "Y")) <= 1e-2
        # the backward ran Cannon's schedule too (reading N7): equal to the oracle's program
        dXc, dWc = cannon.cannon_bwd(grid, shard(grid, spec, dY, "Y"), shard(grid, spec, X, "X"),
                                     shard(grid, spec, W, "W"), 0.5, Fabric())
        assert rel_fro(gather(mode, p, d, spec, per, "dX", "X"), gather_full(grid, spec, dXc, "X")) <= 1e-2
        assert rel_fro(gather(mode, p, d, spec, per, "dW", "W"), gather_full(grid, spec, dWc, "W")) <= 1e-2


def test_cannon_exact_integer_bit_equal(api):
    M, K, N = 144, 216, 216
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    per = tp_layer(api, "2d", 9, 1, M, K, N, X, W, dY, None, "bf16", 0, 0, CANNON)
    spec = spec_of(M, K, N)
    Yr, dXr, dWr, _ = oracle_layer("2d", 9, 1, spec, X, W, dY)
    assert np.array_equal(gather("2d", 9, 1, spec, per, "Y", "Y"), Yr)
    # Cannon's backward: fp32 accumulators on the wire, exact for these integer sums
    assert np.array_equal(gather("2d", 9, 1, spec, per, "dX", "X"), dXr)
    assert np.array_equal(gather("2d", 9, 1, spec, per, "dW", "W"), dWr)
