"""A pre-LN Transformer block on one rank of a tensor-parallel grid, driven through the C ABI
("the rest of the Transformer block in 2D/3D layouts ... then full ViT-S
(C4) and GPT (C5) blocks end to end"). Orchestration only: every step is a library kernel.

    a = LN1(x); qkv = a Wqkv + bqkv; o = MHA(qkv); h1 = x + o Wo + bo;
    c = LN2(h1); f = gelu(c W1 + b1); out = h1 + f W2 + b2                (oracle/block.py)

Layer layouts chain without re-layout: QKV and fc1 are "layer 0" (1D column split / 3D parity
0), the output projection and fc2 "layer 1" (1D row split / parity 1), so their outputs come
back in x's layout (the X block of the QKV layer), which is also the layout of both LayerNorms.
Heads are whole column blocks of the QKV output (tp_attention_*), so the block needs
heads % (column split) == 0 and whole sequences per row block.
"""
from __future__ import annotations

import math

import numpy as np
import torch

from . import api


class TPBlock:
    def __init__(self, grid, M, h, heads, seq, F=None, dtype="bf16", eps=1e-5, flags=0):
        F = F or 4 * h
        self.g, self.M, self.h, self.F, self.heads, self.seq = grid, M, h, F, heads, seq
        self.dtype, self.eps = dtype, eps
        self.tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        D = lambda K, N, layer, extra=0: api.desc(M, K, N, dtype, split_1d=layer, parity_3d=layer,
                                                  flags=flags | extra)
        self.dq, self.dp = D(h, 3 * h, 0), D(h, h, 1)
        self.d1, self.d2 = D(h, F, 0, api.TP_FLAG_GELU), D(F, h, 1)
        mk = lambda d, t: self._alloc(d, t)
        ex = api.tp_shard_extent(grid, self.dq, "X")
        self.ln_cols = (ex[2], ex[3])
        vec = lambda: torch.empty(ex[3], device="cuda", dtype=self.tdt)
        # parameters
        self.W = {"qkv": mk(self.dq, "W"), "o": mk(self.dp, "W"), "1": mk(self.d1, "W"),
                  "2": mk(self.d2, "W")}
        self.b = {"qkv": mk(self.dq, "B")[0], "o": mk(self.dp, "B")[0], "1": mk(self.d1, "B")[0],
                  "2": mk(self.d2, "B")[0]}
        self.ln = {"g1": vec(), "be1": vec(), "g2": vec(), "be2": vec()}
        # activations (x, h1, out, a, c share x's layout)
        self.x, self.a, self.h1, self.c, self.out = (mk(self.dq, "X") for _ in range(5))
        self.qkv, self.o = mk(self.dq, "Y"), mk(self.dp, "X")
        self.y1, self.f, self.y2 = mk(self.dp, "Y"), mk(self.d1, "Y"), mk(self.d2, "Y")
        rows = ex[1]
        # attention row log-sum-exp (fused forward -> fused backward): heads_local x rows
        self.lse = torch.empty(self.qkv.shape[1] // (3 * (h // heads)) * rows, device="cuda",
                               dtype=torch.float32)
        self.st1 = torch.empty(rows, 2, device="cuda", dtype=torch.float32)
        self.st2 = torch.empty_like(self.st1)
        # gradients
        self.dW = {k: torch.empty_like(v) for k, v in self.W.items()}
        self.db = {k: torch.empty_like(v) for k, v in self.b.items()}
        self.dln = {k: torch.empty_like(v) for k, v in self.ln.items()}
        self.dout, self.dx = mk(self.dq, "X"), mk(self.dq, "X")
        self.df, self.dc, self.dh1, self.dt = mk(self.d1, "Y"), mk(self.d1, "X"), mk(self.dq, "X"), mk(self.dq, "X")
        self.do, self.dqkv, self.da = mk(self.dp, "X"), mk(self.dq, "Y"), mk(self.dq, "X")
        # workspaces
        sizes = [api.tp_workspace_size(grid, d) for d in (self.dq, self.dp, self.d1, self.d2)]
        wsb = max([s[0] for s in sizes] + [api.tp_layernorm_ws_size(grid, self.dq, "X"),
                                          api.tp_attention_ws_size(grid, self.dq, seq, heads), 256])
        self.ws = torch.empty(wsb, device="cuda", dtype=torch.uint8)
        self.sv = [torch.empty(max(s[1], 256), device="cuda", dtype=torch.uint8) for s in sizes]

    def _alloc(self, d, t):
        e = api.tp_shard_extent(self.g, d, t)
        return torch.empty(e[1], e[3], device="cuda", dtype=self.tdt)

    # ---- parameters
    def load(self, P):
        """Global fp parameters (numpy, oracle/block.py names) -> this rank's shards."""
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda().to(self.tdt)
        for k, d, key in (("qkv", self.dq, "qkv"), ("o", self.dp, "o"), ("1", self.d1, "1"),
                          ("2", self.d2, "2")):
            api.tp_pack(self.g, d, "W", dev(P["W_" + key]), self.W[k])
            api.tp_pack(self.g, d, "B", dev(P["b_" + key][None, :])[0].contiguous(), self.b[k])
        c0, n = self.ln_cols
        for k in self.ln:
            self.ln[k].copy_(dev(P[k][None, c0:c0 + n])[0])

    def fill(self, seed=42):
        """Seeded synthetic parameters and input (library generator; Xavier-uniform weights)."""
        for i, (k, d) in enumerate((("qkv", self.dq), ("o", self.dp), ("1", self.d1), ("2", self.d2))):
            r0, rows, c0, cols = api.tp_shard_extent(self.g, d, "W")
            api.tp_fill(self.W[k], self.dtype, rows, cols, cols, seed, 16 * i + 1, "uniform",
                        math.sqrt(6.0 / (d.K + d.N)), r0, c0, d.N)
            self.b[k].zero_()
        for k in self.ln:
            (self.ln[k].fill_(1.0) if k.startswith("g") else self.ln[k].zero_())
        r0, rows, c0, cols = api.tp_shard_extent(self.g, self.dq, "X")
        api.tp_fill(self.x, self.dtype, rows, cols, cols, seed, 0, "uniform", 1.0, r0, c0, self.h)
        r0, rows, c0, cols = api.tp_shard_extent(self.g, self.dq, "X")
        api.tp_fill(self.dout, self.dtype, rows, cols, cols, seed, 2, "uniform", 1.0, r0, c0, self.h)

    # ---- forward / backward
    def forward(self):
        g, ws, sv = self.g, self.ws, self.sv
        api.tp_layernorm_fwd(g, self.dq, "X", self.eps, self.x, self.ln["g1"], self.ln["be1"], self.a,
                             self.st1, ws)
        api.tp_linear_fwd(g, self.dq, self.a, self.W["qkv"], self.b["qkv"], self.qkv, sv[0], ws)
        api.tp_attention_fwd(g, self.dq, self.seq, self.heads, self.qkv, self.o, ws, lse=self.lse)
        api.tp_linear_fwd(g, self.dp, self.o, self.W["o"], self.b["o"], self.y1, sv[1], ws)
        api.tp_add(self.x, self.y1, self.h1)
        api.tp_layernorm_fwd(g, self.dq, "X", self.eps, self.h1, self.ln["g2"], self.ln["be2"], self.c,
                             self.st2, ws)
        api.tp_linear_fwd(g, self.d1, self.c, self.W["1"], self.b["1"], self.f, sv[2], ws)
        api.tp_linear_fwd(g, self.d2, self.f, self.W["2"], self.b["2"], self.y2, sv[3], ws)
        api.tp_add(self.h1, self.y2, self.out)

    def backward(self):
        g, ws, sv = self.g, self.ws, self.sv
        api.tp_linear_bwd(g, self.d2, self.dout, self.f, self.W["2"], sv[3], self.df, self.dW["2"],
                          self.db["2"], ws)
        api.tp_linear_bwd(g, self.d1, self.df, self.c, self.W["1"], sv[2], self.dc, self.dW["1"],
                          self.db["1"], ws)
        api.tp_layernorm_bwd(g, self.dq, "X", self.dc, self.h1, self.ln["g2"], self.st2, self.dt,
                             self.dln["g2"], self.dln["be2"], ws)
        api.tp_add(self.dout, self.dt, self.dh1)
        api.tp_linear_bwd(g, self.dp, self.dh1, self.o, self.W["o"], sv[1], self.do, self.dW["o"],
                          self.db["o"], ws)
        api.tp_attention_bwd(g, self.dq, self.seq, self.heads, self.qkv, self.do, self.dqkv, ws,
                             out=self.o, lse=self.lse)
        api.tp_linear_bwd(g, self.dq, self.dqkv, self.a, self.W["qkv"], sv[0], self.da,
                          self.dW["qkv"], self.db["qkv"], ws)
        api.tp_layernorm_bwd(g, self.dq, "X", self.da, self.x, self.ln["g1"], self.st1, self.dt,
                             self.dln["g1"], self.dln["be1"], ws)
        api.tp_add(self.dh1, self.dt, self.dx)

    def step(self):
        self.forward()
        self.backward()

    def flops(self):
        """GEMM flops of one fwd+bwd (6 M K N per linear) + attention (3 x 4 s^2 d per head
        and sequence: QK^T, PV forward; recompute + 4 products backward)."""
        lin = 6.0 * self.M * self.h * (3 * self.h + self.h + 2 * self.F)
        att = (self.M // self.seq) * self.heads * (4 + 10) * self.seq * self.seq * (self.h // self.heads)
        return lin + att
