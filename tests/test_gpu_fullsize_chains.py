"""Parity of the two-layer chains of BASELINE.json configs[3] (ViT-S/16 MLP: 384 -> 1536 -> 384
over 197 tokens x 4096 images = 806,912 rows) and configs[4] (GPT MLP: 8192 -> 32768 -> 8192
over 8 x 2048 = 16,384 tokens) at their FULL sizes, as bench.py --workload c4 / c5 runs them, on
the grids the configs name (C4: 2D q=2 and 3D l=2, plus 1D p=1; C5: 3D l=2 vs 1D p=1), in-process
ranks on one GPU. Expected values: oracle/sampled.chain2_grids (fp64 from the quantised
inputs), tile-stratified samples (one entry per 128 x 128 output tile) with the bars of
test_gpu_c3head.py (relative Frobenius <= 1e-2, every entry within 5e-2 x rms)."""
import numpy as np
import pytest
import torch

import synth
from oracle import sampled

from test_gpu_c3head import check, sampled_outputs_cfg

pytestmark = pytest.mark.gpu

CONFIGS = {"c4": (4096 * 197, [(384, 1536), (1536, 384)]),
           "c5": (16384, [(8192, 32768), (32768, 8192)])}
GRIDS = [("c4", "1d", 1, 1), ("c4", "2d", 4, 1), ("c4", "3d", 8, 1),
         ("c5", "1d", 1, 1), ("c5", "3d", 8, 1)]
_REF = {}


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def expected(name):
    if name not in _REF:
        M, layers = CONFIGS[name]
        (K, H), (_, N) = layers
        X = synth.tensor(42, synth.layer_tid(0, synth.TID_X), M, K)
        W1 = synth.tensor(42, synth.layer_tid(0, synth.TID_W), K, H, scale=synth.xavier_scale(K, H))
        W2 = synth.tensor(42, synth.layer_tid(1, synth.TID_W), H, N, scale=synth.xavier_scale(H, N))
        dY = synth.tensor(42, synth.layer_tid(1, synth.TID_DY), M, N)
        dims = {"Y": (M, N), "dX": (M, K), "dW1": (K, H), "dW2": (H, N)}
        idx = {k: (sampled.stratified_indices(200 + 2 * n, r), sampled.stratified_indices(201 + 2 * n, c))
               for n, (k, (r, c)) in enumerate(dims.items())}
        _REF[name] = (idx, sampled.chain2_grids(X, W1, W2, dY, idx))
        del X, W1, W2, dY
    return _REF[name]


@pytest.mark.parametrize("cfg,mode,p,d", GRIDS, ids=[f"{c}-{m}-p{p}" for c, m, p, _ in GRIDS])
def test_full_size_two_layer_chain(api, cfg, mode, p, d):
    M, layers = CONFIGS[cfg]
    idx, ref = expected(cfg)
    got = sampled_outputs_cfg(api, mode, p, d, 0, idx, M, layers)
    check(got, ref)
