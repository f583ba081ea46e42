"""Pin of the Transformer-block oracle (oracle/block.py): the composition of the separately
pinned pieces equals torch fp64 autograd of the same block written with torch.nn.functional."""
import numpy as np
import torch

import synth
from oracle import block


def params(seed, h, F, heads):
    rnd = lambda t, r, c, s: synth.tensor(seed, t, r, c, dtype="fp32").astype(np.float64) * s
    return {"W_qkv": rnd(0, h, 3 * h, 0.1), "b_qkv": rnd(1, 1, 3 * h, 0.1)[0],
            "W_o": rnd(2, h, h, 0.1), "b_o": rnd(3, 1, h, 0.1)[0],
            "W_1": rnd(4, h, F, 0.1), "b_1": rnd(5, 1, F, 0.1)[0],
            "W_2": rnd(6, F, h, 0.1), "b_2": rnd(7, 1, h, 0.1)[0],
            "g1": 1 + rnd(8, 1, h, 0.1)[0], "be1": rnd(9, 1, h, 0.1)[0],
            "g2": 1 + rnd(10, 1, h, 0.1)[0], "be2": rnd(11, 1, h, 0.1)[0]}


def torch_block(x, P, seq, heads, eps=1e-5):
    h = x.shape[1]
    d = h // heads
    a = torch.nn.functional.layer_norm(x, (h,), P["g1"], P["be1"], eps)
    qkv = a @ P["W_qkv"] + P["b_qkv"]
    B = x.shape[0] // seq
    t = qkv.reshape(B, seq, heads, 3, d)
    q, k, v = (t[:, :, :, i].permute(0, 2, 1, 3) for i in range(3))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v).permute(0, 2, 1, 3).reshape(B * seq, h)
    h1 = x + o @ P["W_o"] + P["b_o"]
    c = torch.nn.functional.layer_norm(h1, (h,), P["g2"], P["be2"], eps)
    f = torch.nn.functional.gelu(c @ P["W_1"] + P["b_1"])
    return h1 + f @ P["W_2"] + P["b_2"]


def test_block_matches_torch_autograd():
    seq, heads, dh, F = 16, 2, 8, 64
    h = heads * dh
    M = 2 * seq
    P = params(3, h, F, heads)
    x = synth.tensor(3, 20, M, h, dtype="fp32").astype(np.float64)
    dout = synth.tensor(3, 21, M, h, dtype="fp32").astype(np.float64)
    out, S = block.block_fwd(x, P, seq, heads)
    G = block.block_bwd(dout, P, S, seq, heads)
    tP = {k: torch.tensor(v, requires_grad=True) for k, v in P.items()}
    tx = torch.tensor(x, requires_grad=True)
    ref = torch_block(tx, tP, seq, heads)
    assert np.allclose(out, ref.detach().numpy(), atol=1e-11)
    ref.backward(torch.tensor(dout))
    assert np.allclose(G["x"], tx.grad.numpy(), atol=1e-10)
    for k in P:
        assert np.allclose(G[k], tP[k].grad.numpy(), atol=1e-10), k
