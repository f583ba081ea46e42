"""Multi-head self-attention core between the QKV and output projections of a Transformer
block, as laid out by the tensor-parallel linears. TEST INFRASTRUCTURE ONLY.

SURVEY 8(f) NEXT-2: "attention core with heads split across columns" (P:L309 parallelized
components; P:L445 ViT blocks; the attention formula P:L604). Reading N5:

* tokens are rows of the activation [M = batch x seq, h]; the QKV linear (h -> 3h) puts head g
  in columns [3 d g, 3 d (g+1)) as [q | k | v] (d = h / heads), so a column block of the QKV
  output holds whole heads and a row block whole sequences when its row extent is a multiple
  of seq -> every head and sequence is local: no communication in any TP mode;
* per sequence b and head g: O = softmax(Q K^T scale) V (scale 1/sqrt(d) by default), written
  to columns [d g, d (g+1)) of the output [M, h] -- the layout of the output projection's input.
"""
from __future__ import annotations

import math

import numpy as np

from . import ring_attention as ra


def _split(qkv, seq, heads):
    qkv = np.asarray(qkv, np.float64)
    M, n3 = qkv.shape
    d = n3 // (3 * heads)
    B = M // seq
    # [B, seq, heads, 3, d]
    return qkv.reshape(B, seq, heads, 3, d), B, d


def mha_fwd(qkv, seq, heads, scale=None):
    x, B, d = _split(qkv, seq, heads)
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    out = np.zeros((B, seq, heads, d))
    for b in range(B):
        for g in range(heads):
            out[b, :, g, :] = ra.attention(x[b, :, g, 0], x[b, :, g, 1], x[b, :, g, 2], scale)[0]
    return out.reshape(B * seq, heads * d)


def mha_bwd(qkv, dout, seq, heads, scale=None):
    """d(qkv) for dL/d(out) = dout (same layouts as mha_fwd)."""
    x, B, d = _split(qkv, seq, heads)
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    do = np.asarray(dout, np.float64).reshape(B, seq, heads, d)
    g_ = np.zeros_like(x)
    for b in range(B):
        for g in range(heads):
            dq, dk, dv = ra.attention_bwd(x[b, :, g, 0], x[b, :, g, 1], x[b, :, g, 2], do[b, :, g], scale)
            g_[b, :, g, 0], g_[b, :, g, 1], g_[b, :, g, 2] = dq, dk, dv
    return g_.reshape(B * seq, heads * 3 * d)
