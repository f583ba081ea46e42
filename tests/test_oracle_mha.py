"""Pins of the multi-head attention core oracle (oracle/mha.py): torch fp64
scaled_dot_product_attention and its autograd on the same head / column layout."""
import numpy as np
import torch

import synth
from oracle import mha


def test_mha_matches_torch_sdpa_and_autograd():
    B, seq, heads, d = 2, 16, 3, 8
    qkv = synth.tensor(4, 0, B * seq, 3 * heads * d, dtype="fp32").astype(np.float64)
    dout = synth.tensor(4, 1, B * seq, heads * d, dtype="fp32").astype(np.float64)
    t = torch.tensor(qkv, requires_grad=True)
    x = t.reshape(B, seq, heads, 3, d)
    q, k, v = (x[:, :, :, i].permute(0, 2, 1, 3) for i in range(3))   # [B, heads, seq, d]
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v)      # [B, heads, seq, d]
    o = o.permute(0, 2, 1, 3).reshape(B * seq, heads * d)
    assert np.allclose(mha.mha_fwd(qkv, seq, heads), o.detach().numpy(), atol=1e-12)
    o.backward(torch.tensor(dout))
    assert np.allclose(mha.mha_bwd(qkv, dout, seq, heads), t.grad.numpy(), atol=1e-12)


def test_heads_are_independent_column_blocks():
    """Changing head 1's q/k/v columns leaves head 0's output columns unchanged."""
    seq, heads, d = 8, 2, 4
    qkv = synth.tensor(5, 0, seq, 3 * heads * d, dtype="fp32").astype(np.float64)
    a = mha.mha_fwd(qkv, seq, heads)
    qkv2 = qkv.copy()
    qkv2[:, 3 * d:] += 1.0
    b = mha.mha_fwd(qkv2, seq, heads)
    assert np.array_equal(a[:, :d], b[:, :d]) and not np.allclose(a[:, d:], b[:, d:])
