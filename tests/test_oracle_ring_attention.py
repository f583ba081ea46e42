"""Pins of the Ring Self-Attention oracle (oracle/ring_attention.py): the SPEC's worked
examples (tests/golden/rsa_examples.json), torch fp64 scaled_dot_product_attention
(library routine), a pure-Python softmax on a tiny case, the volume law, row-stochasticity,
parallel-degree invariance and V = 0."""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import ring_attention as rsa
from oracle.fabric import Ledger


def qkv(seed, s, d):
    return (synth.tensor(seed, 0, s, d, dtype="fp32").astype(np.float64),
            synth.tensor(seed, 1, s, d, dtype="fp32").astype(np.float64),
            synth.tensor(seed, 2, s, d, dtype="fp32").astype(np.float64))


def gathered(out, N):
    return np.concatenate([out[r] for r in range(N)], axis=0)


def test_golden_examples():
    import json
    import os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "rsa_examples.json")))
    e = g["examples"][0]
    Q, K, V = qkv(e["seed"], e["s"], e["d_k"])
    led = Ledger()
    out, _ = rsa.ring_attention(rsa.shards(Q, 1), rsa.shards(K, 1), rsa.shards(V, 1), ledger=led)
    ref, _ = rsa.attention(Q, K, V)
    assert np.allclose(out[0], ref, atol=1e-14) and led.total() == e["volume"]
    e = g["examples"][1]
    Q, K, V = qkv(e["seed"], e["s"], e["d_k"])
    _, S = rsa.ring_attention(rsa.shards(Q, 2), rsa.shards(K, 2), rsa.shards(V, 2))
    serial = (Q @ K.T) / math.sqrt(e["d_k"])
    assert np.allclose(gathered(S, 2), serial, atol=e["score_tol"], rtol=0)
    e = g["examples"][2]
    Q, K, V = qkv(e["seed"], e["s"], e["d_k"])
    out, _ = rsa.ring_attention(rsa.shards(Q, 4), rsa.shards(K, 4), rsa.shards(V, 4))
    assert np.allclose(gathered(out, 4), rsa.attention(Q, K, V)[0], atol=e["out_tol"], rtol=0)
    e = g["examples"][3]
    Q, K, V = qkv(e["seed"], e["s"], e["d_k"])
    o2 = gathered(rsa.ring_attention(rsa.shards(Q, 2), rsa.shards(K, 2), rsa.shards(V, 2))[0], 2)
    o4 = gathered(rsa.ring_attention(rsa.shards(Q, 4), rsa.shards(K, 4), rsa.shards(V, 4))[0], 4)
    assert np.allclose(o2, o4, atol=e["tol"], rtol=0)


def test_matches_torch_sdpa():
    Q, K, V = qkv(7, 64, 16)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(Q)[None, None], torch.tensor(K)[None, None], torch.tensor(V)[None, None])[0, 0]
    out, _ = rsa.ring_attention(rsa.shards(Q, 4), rsa.shards(K, 4), rsa.shards(V, 4))
    assert np.allclose(gathered(out, 4), ref.numpy(), atol=1e-12, rtol=0)


def test_python_loop_softmax_tiny():
    Q, K, V = qkv(11, 4, 2)
    out, _ = rsa.ring_attention(rsa.shards(Q, 2), rsa.shards(K, 2), rsa.shards(V, 2))
    full = gathered(out, 2)
    for i in range(4):
        sc = [sum(Q[i][c] * K[j][c] for c in range(2)) / math.sqrt(2) for j in range(4)]
        m = max(sc)
        w = [math.exp(x - m) for x in sc]
        z = sum(w)
        for c in range(2):
            assert abs(full[i][c] - sum(w[j] / z * V[j][c] for j in range(4))) < 1e-13


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_volume_law_and_row_stochastic(N):
    s, d = 16, 8
    Q, K, V = qkv(2, s, d)
    led = Ledger()
    out, S = rsa.ring_attention(rsa.shards(Q, N), rsa.shards(K, N), rsa.shards(V, N), ledger=led)
    assert led.total() == 2 * (N - 1) * s * d
    assert led.total("ring_k") == (N - 1) * N * (s // N) * d
    A = rsa.attention(Q, K, V)[1]
    assert np.allclose(A.sum(axis=1), 1.0, atol=1e-12)


def test_zero_values_and_indivisible():
    Q, K, V = qkv(4, 8, 4)
    out, _ = rsa.ring_attention(rsa.shards(Q, 2), rsa.shards(K, 2), rsa.shards(0 * V, 2))
    assert not gathered(out, 2).any()
    with pytest.raises(rsa.IndivisibleSequence):
        rsa.shards(Q, 3)


def test_backward_matches_torch_autograd_and_ring():
    Q, K, V = qkv(13, 32, 8)
    dO = synth.tensor(13, 3, 32, 8, dtype="fp32").astype(np.float64)
    tq, tk, tv = (torch.tensor(a, requires_grad=True) for a in (Q, K, V))
    out = torch.nn.functional.scaled_dot_product_attention(tq[None, None], tk[None, None], tv[None, None])[0, 0]
    out.backward(torch.tensor(dO))
    dQ, dK, dV = rsa.attention_bwd(Q, K, V, dO)
    assert np.allclose(dQ, tq.grad.numpy(), atol=1e-12)
    assert np.allclose(dK, tk.grad.numpy(), atol=1e-12)
    assert np.allclose(dV, tv.grad.numpy(), atol=1e-12)
    for N in (1, 2, 4):
        rq, rk, rv = rsa.ring_attention_bwd(rsa.shards(Q, N), rsa.shards(K, N), rsa.shards(V, N),
                                            rsa.shards(dO, N))
        assert np.allclose(gathered(rq, N), dQ, atol=1e-12)
        assert np.allclose(gathered(rk, N), dK, atol=1e-12)
        assert np.allclose(gathered(rv, N), dV, atol=1e-12)


def test_backward_finite_differences():
    Q, K, V = qkv(17, 8, 4)
    dO = synth.tensor(17, 3, 8, 4, dtype="fp32").astype(np.float64)
    dQ, dK, dV = rsa.attention_bwd(Q, K, V, dO)
    loss = lambda Q_, K_, V_: float((rsa.attention(Q_, K_, V_)[0] * dO).sum())
    h = 1e-6
    for A, G, which in ((Q, dQ, 0), (K, dK, 1), (V, dV, 2)):
        E = np.zeros_like(A)
        E[3, 1] = h
        args_p = [Q, K, V]
        args_m = [Q, K, V]
        args_p[which] = A + E
        args_m[which] = A - E
        assert abs((loss(*args_p) - loss(*args_m)) / (2 * h) - G[3, 1]) < 1e-7
