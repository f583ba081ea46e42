"""A pre-LN Transformer block in the tensor-parallel layouts ("full ViT-S
(C4) and GPT (C5) blocks end to end"). TEST INFRASTRUCTURE ONLY.

The block (ViT; GPT-style; reading N6) composed from the pinned pieces:

    a   = LN1(x)
    qkv = a . Wqkv + bqkv                  (head g: columns [3 d g, 3 d (g+1)) = [q | k | v])
    o   = MHA(qkv)                         (oracle/mha.py)
    h1  = x + o . Wo + bo
    c   = LN2(h1)
    f   = gelu(c . W1 + b1)                (oracle/activation.py)
    out = h1 + f . W2 + b2

and its backward by the chain rule of those pieces (each piece is pinned separately; the
composition is pinned to torch fp64 autograd in tests/test_oracle_block.py).
"""
from __future__ import annotations

import numpy as np

from . import activation as act
from . import dense, mha
from . import layernorm as ln


def block_fwd(x, P, seq, heads, eps=1e-5):
    """P: dict of W_qkv, b_qkv, W_o, b_o, W_1, b_1, W_2, b_2, g1, be1, g2, be2 (fp64 arrays)."""
    x = np.asarray(x, np.float64)
    a, mu1, r1 = ln.ln_fwd(x, P["g1"], P["be1"], eps)
    qkv = dense.linear_fwd(a, P["W_qkv"], P["b_qkv"])
    o = mha.mha_fwd(qkv, seq, heads)
    h1 = x + dense.linear_fwd(o, P["W_o"], P["b_o"])
    c, mu2, r2 = ln.ln_fwd(h1, P["g2"], P["be2"], eps)
    z = dense.linear_fwd(c, P["W_1"], P["b_1"])
    f = act.gelu(z)
    out = h1 + dense.linear_fwd(f, P["W_2"], P["b_2"])
    saved = dict(x=x, a=a, mu1=mu1, r1=r1, qkv=qkv, o=o, h1=h1, c=c, mu2=mu2, r2=r2, z=z, f=f)
    return out, saved


def block_bwd(dout, P, S, seq, heads):
    """Gradients of every input and parameter of block_fwd (dict)."""
    G = {}
    dout = np.asarray(dout, np.float64)
    df, G["W_2"], G["b_2"] = dense.linear_bwd(dout, S["f"], P["W_2"])
    dz = df * act.gelu_grad(S["z"])
    dc, G["W_1"], G["b_1"] = dense.linear_bwd(dz, S["c"], P["W_1"])
    dh1_ln, G["g2"], G["be2"] = ln.ln_bwd(dc, S["h1"], P["g2"], S["mu2"], S["r2"])
    dh1 = dout + dh1_ln
    do, G["W_o"], G["b_o"] = dense.linear_bwd(dh1, S["o"], P["W_o"])
    dqkv = mha.mha_bwd(S["qkv"], do, seq, heads)
    da, G["W_qkv"], G["b_qkv"] = dense.linear_bwd(dqkv, S["a"], P["W_qkv"])
    dx_ln, G["g1"], G["be1"] = ln.ln_bwd(da, S["x"], P["g1"], S["mu1"], S["r1"])
    G["x"] = dh1 + dx_ln
    return G
