"""A chain of tensor-parallel linear layers on one rank — the paper's range-test model
("a model which consists of two linear layers") — driven through the C ABI.

Orchestration only: allocates this rank's shards (torch device memory), fills them with the
library's seeded generator (tp_fill), and calls tp_linear_fwd / tp_linear_bwd layer by layer.
Layer i uses split_1d = parity_3d = i % 2, so layer i's Y layout is layer i+1's X layout
(1D column -> row, 3D parity 0 -> 1; 2D/2.5D are layout-preserving): no re-layout between
layers. Inputs follow the synth recipe: X = tensor(seed, layer_tid(0, X)), W_i = Xavier
tensor(seed, layer_tid(i, W)), dY of the last layer = tensor(seed, layer_tid(L-1, dY)).
"""
from __future__ import annotations

import math

import torch

from . import api

TID_X, TID_W, TID_DY = 0, 1, 2


def layer_tid(layer, tid):
    return 16 * layer + tid


class TPMLP:
    def __init__(self, grid, M, layers, dtype="bf16", seed=42, flags=0, alpha=1.0,
                 kind="uniform", fill=True, act=None):
        self.g, self.M, self.layers, self.dtype, self.seed = grid, M, list(layers), dtype, seed
        self.tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        self.kind = kind
        # act="gelu": GeLU after every even layer (fc1 of each fc1 -> gelu -> fc2 pair)
        gelu = lambda i: api.TP_FLAG_GELU if act == "gelu" and i % 2 == 0 and i + 1 < len(layers) else 0
        self.descs = [api.desc(M, K, N, dtype, split_1d=i % 2, parity_3d=i % 2,
                               flags=flags | gelu(i), alpha=alpha)
                      for i, (K, N) in enumerate(self.layers)]
        L = len(self.layers)
        self.x = self._alloc(0, "X")
        self.W = [self._alloc(i, "W") for i in range(L)]
        self.Y = [self._alloc(i, "Y") for i in range(L)]
        self.dY = self._alloc(L - 1, "Y")
        self.dX = [torch.empty_like(self.x)] + [torch.empty_like(self.Y[i]) for i in range(L - 1)]
        self.dW = [torch.empty_like(w) for w in self.W]
        sizes = [api.tp_workspace_size(self.g, d) for d in self.descs]
        self.ws = torch.empty(max(max(s[0] for s in sizes), 256), device="cuda", dtype=torch.uint8)
        self.saved = [torch.empty(s[1], device="cuda", dtype=torch.uint8) if s[1] else None
                      for s in sizes]
        if flags & api.TP_FLAG_PEER_FUSED:
            # every tensor a peer may read is a symmetric registered buffer (collective, same
            # order on all ranks): layer inputs X / Y_i, weights W_i, gradients dY / dX_i
            # (and the workspace: the fused 1D reduce-scatter's receive slots live in it)
            for t in [self.x, *self.W, *self.Y, self.dY, *self.dX, self.ws]:
                api.tp_register_buffer(self.g, t)
        if fill:
            self.fill_inputs()

    def _ext(self, i, t):
        return api.tp_shard_extent(self.g, self.descs[i], t)

    def _alloc(self, i, t):
        e = self._ext(i, t)
        return torch.empty(e[1], e[3], device="cuda", dtype=self.tdt)

    def _fill(self, buf, i, t, tid, scale):
        r0, rows, c0, cols = self._ext(i, t)
        d = self.descs[i]
        gcols = {"X": d.K, "W": d.N, "Y": d.N}[t]
        api.tp_fill(buf, self.dtype, rows, cols, cols, self.seed, tid, self.kind, scale, r0, c0,
                    gcols)

    def fill_inputs(self):
        L = len(self.layers)
        self._fill(self.x, 0, "X", layer_tid(0, TID_X), 1.0)
        for i, (K, N) in enumerate(self.layers):
            scale = math.sqrt(6.0 / (K + N)) if self.kind == "uniform" else 1.0
            self._fill(self.W[i], i, "W", layer_tid(i, TID_W), scale)
        self._fill(self.dY, L - 1, "Y", layer_tid(L - 1, TID_DY), 1.0)

    def forward(self):
        inp = self.x
        for i, d in enumerate(self.descs):
            api.tp_linear_fwd(self.g, d, inp, self.W[i], None, self.Y[i], self.saved[i], self.ws)
            inp = self.Y[i]

    def backward(self):
        dy = self.dY
        for i in reversed(range(len(self.descs))):
            x = self.x if i == 0 else self.Y[i - 1]
            api.tp_linear_bwd(self.g, self.descs[i], dy, x, self.W[i], self.saved[i], self.dX[i],
                              self.dW[i], None, self.ws)
            dy = self.dX[i]

    def step(self):
        self.forward()
        self.backward()

    def flops(self):
        return sum(6.0 * self.M * K * N for K, N in self.layers)
