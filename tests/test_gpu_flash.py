"""The fused attention forward (flash.cu; scores kept on chip, online softmax over key tiles)
through the attention core (tp_attention_fwd, bf16, d in {64, 128}) against the oracle
(oracle/mha.py), including sequences that are not a multiple of the 128-key tile, and against
the two-pass path (TP_FLASH=0) in a child process."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth
from oracle import mha

from tp_harness import rel_fro

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def run_core(api, B, seq, heads, dh, qkv, scale=0.0):
    g = api.tp_grid_init("1d", 1, 0)
    h = heads * dh
    d = api.desc(B * seq, h, 3 * h, "bf16")
    x = torch.from_numpy(qkv.astype(np.float32)).cuda().to(torch.bfloat16)
    out = torch.empty(B * seq, h, device="cuda", dtype=torch.bfloat16)
    ws = torch.empty(api.tp_attention_ws_size(g, d, seq, heads), device="cuda", dtype=torch.uint8)
    api.tp_attention_fwd(g, d, seq, heads, x, out, ws, scale=scale)
    torch.cuda.synchronize()
    api.tp_grid_destroy(g)
    return out.float().cpu().numpy().astype(np.float64)


@pytest.mark.parametrize("seq", [128, 200, 1024, 2048])
@pytest.mark.parametrize("dh", [64, 128])
def test_flash_forward_vs_oracle(api, seq, dh):
    B, heads = 2, 3
    qkv = synth.tensor(41, 0, B * seq, 3 * heads * dh, dtype="bf16").astype(np.float64) * 2.0
    got = run_core(api, B, seq, heads, dh, qkv)
    assert rel_fro(got, mha.mha_fwd(qkv, seq, heads)) <= 1e-2


def test_flash_scale_and_large_scores(api):
    """Explicit scale and scores of magnitude ~30 (the running max must rescale correctly)."""
    B, seq, heads, dh = 1, 512, 2, 64
    qkv = synth.tensor(43, 0, B * seq, 3 * heads * dh, dtype="bf16").astype(np.float64) * 4.0
    got = run_core(api, B, seq, heads, dh, qkv, scale=0.3)
    assert rel_fro(got, mha.mha_fwd(qkv, seq, heads, scale=0.3)) <= 1e-2


def test_flash_matches_two_pass_path():
    code = ("import numpy as np, torch, sys; sys.path.insert(0, 'tests'); import synth;"
            "from test_gpu_flash import run_core; from paper_2110_14883_b200 import api;"
            "q = synth.tensor(47, 0, 2 * 256, 3 * 2 * 64, dtype='bf16').astype(np.float64);"
            "np.save(sys.argv[1], run_core(api, 2, 256, 2, 64, q))")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        path = f"/tmp/flash_cmp_{flag}.npy"
        r = subprocess.run([sys.executable, "-c", code, path], cwd=root, capture_output=True,
                           text=True, timeout=300, env=dict(os.environ, TP_FLASH=flag))
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    assert rel_fro(outs[0], outs[1]) <= 1e-2
