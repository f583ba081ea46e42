"""Parity of the fused peer-panel SUMMA (TP_FLAG_PEER_FUSED) against the
oracle's rank-by-rank program: the same layer results as the collective schedule (a-5 .. a-8),
computed owner-side as ONE multi-panel GEMM per product whose K-panels are read straight from
the owners' registered shards. Ranks are in-process threads on cuda:0 (LOCAL transport), so
"peer memory" is the same GPU's memory; across GPUs the same kernel reads NVLink peer memory
through the IPC-mapped pointers tp_register_buffer exchanges.
"""
import numpy as np
import pytest
import torch

import synth

from tp_harness import gather, oracle_layer, rel_fro, spec_of, tp_layer

pytestmark = pytest.mark.gpu

FUSED = 0x4  # TP_FLAG_PEER_FUSED

# (mode, p, d, M, K, N): per-rank blocks > 128 rows with ragged tails, panels of K not a
# multiple of the 64-wide k-block (the per-panel tensor map zero-fills the tail)
CASES = [
    ("2d", 4, 1, 520, 400, 656, 0),     # q=2: 260 x 200 x 328 blocks
    ("2d", 9, 1, 408, 432, 600, 0),     # q=3: 136 x 144 x 200
    ("2d", 16, 1, 576, 544, 544, 0),    # q=4: 144 x 136 x 136 (four panels per product)
    ("2.5d", 8, 2, 800, 272, 528, 0),   # q=2, d=2 (replicated W): 200 x 136 x 264
    # 3D l=2, both parities: shards [M/4, K/2] [K/4, N/2] [M/4, N/2] = 136 x 288, 144 x 200
    ("3d", 8, 1, 544, 576, 400, 0),
    ("3d", 8, 1, 544, 576, 400, 1),
]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def _id(c):
    return f"{c[0]}-p{c[1]}-d{c[2]}-par{c[6]}"


@pytest.mark.parametrize("case", CASES, ids=_id)
@pytest.mark.parametrize("with_bias", [False, True])
def test_fused_vs_oracle(api, case, with_bias):
    mode, p, d, M, K, N, par = case
    X, W, dY, b = synth.layer_inputs(11, M, K, N, with_bias=True)
    b = b if with_bias else None
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, "bf16", parity=par, flags=FUSED,
                   alpha=0.5)
    spec = spec_of(M, K, N, parity=par)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY, b, alpha=0.5)
    assert rel_fro(gather(mode, p, d, spec, per, "Y", "Y"), Yr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dX", "X"), dXr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dW", "W"), dWr) <= 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "dB", "B"), dbr) <= 1e-2
    # owner computes: the forward is exactly one GEMM launch per rank (no panel copies, no
    # partial-sum passes) — proof the fused path ran rather than the collective schedule
    assert per[0]["n_fwd"] == p


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_fused_exact_integer_bit_equal(api, case):
    """Ternary inputs: every product is an exact small integer (|sum| <= K, M < 2^24) so the
    fused TMEM accumulation must be bit-equal to the oracle (A17)."""
    mode, p, d, M, K, N, par = case
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, None, "bf16", parity=par, flags=FUSED)
    spec = spec_of(M, K, N, parity=par)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY)
    for key, t, ref in (("Y", "Y", Yr), ("dX", "X", dXr), ("dW", "W", dWr), ("dB", "B", dbr)):
        assert np.array_equal(gather(mode, p, d, spec, per, key, t), ref), key


def test_fused_matches_collective_schedule(api):
    """Same inputs, both schedules: results agree to bf16 rounding of differently-ordered fp32
    sums (the collective path rounds each SUMMA partial to bf16; fused rounds once)."""
    mode, p, d, M, K, N, _ = CASES[0]
    X, W, dY, b = synth.layer_inputs(3, M, K, N, with_bias=True)
    a = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, "bf16", flags=FUSED)
    c = tp_layer(api, mode, p, d, M, K, N, X, W, dY, b, "bf16", flags=0)
    spec = spec_of(M, K, N)
    for key, t in (("Y", "Y"), ("dX", "X"), ("dW", "W"), ("dB", "B")):
        assert rel_fro(gather(mode, p, d, spec, a, key, t), gather(mode, p, d, spec, c, key, t)) <= 1e-2
    assert a[0]["n_fwd"] == p and c[0]["n_fwd"] > p


def test_fused_falls_back_on_small_blocks(api):
    """The flag with blocks <= 128 rows (below the CTA-pair tile) takes the collective
    schedule: still correct."""
    M, K, N = 144, 256, 192  # 72-row blocks: below the CTA-pair kernel's tile
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    per = tp_layer(api, "2d", 4, 1, M, K, N, X, W, dY, None, "bf16", flags=FUSED)
    spec = spec_of(M, K, N)
    Yr, dXr, dWr, _ = oracle_layer("2d", 4, 1, spec, X, W, dY)
    assert np.array_equal(gather("2d", 4, 1, spec, per, "Y", "Y"), Yr)
    assert np.array_equal(gather("2d", 4, 1, spec, per, "dX", "X"), dXr)
    assert np.array_equal(gather("2d", 4, 1, spec, per, "dW", "W"), dWr)


@pytest.mark.parametrize("par", [0, 1])
def test_fused_3d_backward_after_unfused_dy(api, par):
    """Fused forward (X, W registered) followed by a backward whose dY is NOT registered: the
    backward falls back to the collective schedule and must first re-gather X and W (the fused
    forward left nothing in `saved`)."""
    import torch
    from tp_harness import run_ranks, to_dev, to_np, TORCH_DT
    M, K, N = 544, 576, 400
    X, W, dY, _ = synth.layer_inputs(7, M, K, N, kind="ternary")
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)
    gX, gW, gdY = to_dev(X, "bf16"), to_dev(W, "bf16"), to_dev(dY, "bf16")
    torch.cuda.synchronize()

    def rank_fn(r):
        g = api.tp_grid_init("3d", 8, r, 0, 1, 0, api.TP_TRANSPORT_LOCAL, uid)
        s = torch.cuda.Stream()
        try:
            with torch.cuda.stream(s):
                ds = api.desc(M, K, N, "bf16", 0, par, FUSED)
                ext = {t: api.tp_shard_extent(g, ds, t) for t in ("X", "W", "Y")}
                mk = lambda t: torch.empty(ext[t][1], ext[t][3], device="cuda", dtype=torch.bfloat16)
                x, w, y, dy = mk("X"), mk("W"), mk("Y"), mk("Y")
                api.tp_register_buffer(g, x)
                api.tp_register_buffer(g, w)
                api.tp_pack(g, ds, "X", gX, x)
                api.tp_pack(g, ds, "W", gW, w)
                api.tp_pack(g, ds, "Y", gdY, dy)
                wsb, svb = api.tp_workspace_size(g, ds)
                ws = torch.empty(max(wsb, 1), device="cuda", dtype=torch.uint8)
                sv = torch.empty(svb, device="cuda", dtype=torch.uint8)
                api.tp_linear_fwd(g, ds, x, w, None, y, sv, ws)
                dx, dw = torch.empty_like(x), torch.empty_like(w)
                api.tp_linear_bwd(g, ds, dy, x, w, sv, dx, dw, None, ws)
            s.synchronize()
            return {"Y": to_np(y), "dX": to_np(dx), "dW": to_np(dw)}
        finally:
            s.synchronize()
            api.tp_grid_destroy(g)

    per = run_ranks(8, rank_fn)
    spec = spec_of(M, K, N, parity=par)
    Yr, dXr, dWr, _ = oracle_layer("3d", 8, 1, spec, X, W, dY)
    for key, t, ref in (("Y", "Y", Yr), ("dX", "X", dXr), ("dW", "W", dWr)):
        assert np.array_equal(gather("3d", 8, 1, spec, per, key, t), ref), key


@pytest.mark.parametrize("p,split", [(2, 0), (4, 0), (8, 0), (2, 1), (4, 1)])
def test_fused_1d_reduce_scatter(api, p, split):
    """1D: the all-reduced product (column split: dX in backward; row split: Y in forward) is
    reduce-scattered by the GEMM epilogue into the owners' receive slots and all-gathered."""
    M, K, N = 512, 384, 640
    X, W, dY, b = synth.layer_inputs(29, M, K, N, with_bias=True)
    per = tp_layer(api, "1d", p, 1, M, K, N, X, W, dY, b, "bf16", split, 0, FUSED, alpha=0.5)
    spec = spec_of(M, K, N, split)
    Yr, dXr, dWr, dbr = oracle_layer("1d", p, 1, spec, X, W, dY, b, alpha=0.5)
    assert rel_fro(gather("1d", p, 1, spec, per, "Y", "Y"), Yr) <= 1e-2
    assert rel_fro(gather("1d", p, 1, spec, per, "dX", "X"), dXr) <= 1e-2
    assert rel_fro(gather("1d", p, 1, spec, per, "dW", "W"), dWr) <= 1e-2
    assert rel_fro(gather("1d", p, 1, spec, per, "dB", "B"), dbr) <= 1e-2
    if split == 1:  # the forward is one GEMM + the sum kernel per rank (+ peer copies)
        assert per[0]["n_fwd"] == 2 * p


def test_fused_1d_exact_integer(api):
    M, K, N = 256, 128, 256
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    for split in (0, 1):
        per = tp_layer(api, "1d", 4, 1, M, K, N, X, W, dY, None, "bf16", split, 0, FUSED)
        spec = spec_of(M, K, N, split)
        Yr, dXr, dWr, _ = oracle_layer("1d", 4, 1, spec, X, W, dY)
        assert np.array_equal(gather("1d", 4, 1, spec, per, "Y", "Y"), Yr)
        assert np.array_equal(gather("1d", 4, 1, spec, per, "dX", "X"), dXr)
        assert np.array_equal(gather("1d", 4, 1, spec, per, "dW", "W"), dWr)


DEPTH_SHARDED = 0x1  # TP_FLAG_W25_DEPTH_SHARDED


@pytest.mark.parametrize("p,d,M,K,N", [
    (8, 2, 800, 544, 528),   # q=2, d=2: blocks 200 x 272 (W shard 136 x 264), four panels
    (4, 4, 600, 544, 520),   # q=1, d=4: blocks 150 x 544 (W shard 136 x 520), four panels
    (8, 2, 528, 1056, 400),  # hq = 264: K-panels not a multiple of the 64-wide k-block
], ids=["q2d2", "q1d4", "q2d2-ragged"])
@pytest.mark.parametrize("with_bias", [False, True])
def test_fused_depth_sharded_25d(api, p, d, M, K, N, with_bias):
    """2.5D with the weight depth-sharded (1/p per rank): every product is one multi-panel GEMM
    whose q*d K-panels are the depth pieces of the SUMMA panels, read from their owners; no depth
    all-gather of W, no depth reduce-scatter of dW."""
    X, W, dY, b = synth.layer_inputs(17, M, K, N, with_bias=True)
    b = b if with_bias else None
    fl = FUSED | DEPTH_SHARDED
    per = tp_layer(api, "2.5d", p, d, M, K, N, X, W, dY, b, "bf16", flags=fl, alpha=0.5)
    spec = spec_of(M, K, N, flags=fl)
    Yr, dXr, dWr, dbr = oracle_layer("2.5d", p, d, spec, X, W, dY, b, alpha=0.5)
    assert rel_fro(gather("2.5d", p, d, spec, per, "Y", "Y"), Yr) <= 1e-2
    assert rel_fro(gather("2.5d", p, d, spec, per, "dX", "X"), dXr) <= 1e-2
    assert rel_fro(gather("2.5d", p, d, spec, per, "dW", "W"), dWr) <= 1e-2
    if with_bias:
        assert rel_fro(gather("2.5d", p, d, spec, per, "dB", "B"), dbr) <= 1e-2
    assert per[0]["n_fwd"] == p  # one GEMM per rank: the fused path ran


def test_fused_depth_sharded_25d_exact_integer(api):
    M, K, N = 544, 544, 272
    X, W, dY, _ = synth.layer_inputs(6, M, K, N, kind="ternary")
    fl = FUSED | DEPTH_SHARDED
    per = tp_layer(api, "2.5d", 8, 2, M, K, N, X, W, dY, None, "bf16", flags=fl)
    spec = spec_of(M, K, N, flags=fl)
    Yr, dXr, dWr, _ = oracle_layer("2.5d", 8, 2, spec, X, W, dY)
    assert np.array_equal(gather("2.5d", 8, 2, spec, per, "Y", "Y"), Yr)
    assert np.array_equal(gather("2.5d", 8, 2, spec, per, "dX", "X"), dXr)
    assert np.array_equal(gather("2.5d", 8, 2, spec, per, "dW", "W"), dWr)


STAGED = 0x40  # TP_FLAG_PEER_STAGED


@pytest.mark.parametrize("case", CASES, ids=_id)
def test_fused_staged_exact_integer_bit_equal(api, case):
    """TP_FLAG_PEER_STAGED: every peer shard a panel GEMM reads is first pulled once by the copy
    engine into local workspace (the path taken automatically for peers on another GPU). Same
    products, so bit-equal on exact-integer inputs; the forward is still one GEMM launch."""
    mode, p, d, M, K, N, par = case
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    per = tp_layer(api, mode, p, d, M, K, N, X, W, dY, None, "bf16", parity=par, flags=FUSED | STAGED)
    spec = spec_of(M, K, N, parity=par)
    Yr, dXr, dWr, dbr = oracle_layer(mode, p, d, spec, X, W, dY)
    for key, t, ref in (("Y", "Y", Yr), ("dX", "X", dXr), ("dW", "W", dWr), ("dB", "B", dbr)):
        assert np.array_equal(gather(mode, p, d, spec, per, key, t), ref), key
    assert per[0]["n_fwd"] == p
    assert all(r["staged_fwd"] > 0 and r["staged_bwd"] > 0 for r in per)


def test_fused_staged_bytes_equal_summa_volume(api):
    """2D q=2: staged, each rank pulls exactly the distinct peer shards its panels need, once -
    in the forward X[i,t] (t != j) and W[t,j] (t != i): the bytes SUMMA's broadcasts deliver; the
    backward's owner-computes products need dY[i,t], W[j,t], X[t,i], dY[t,j] (deduplicated)."""
    M, K, N = 520, 400, 656
    q = 2
    mb, kq, nq = M // q, K // q, N // q
    X, W, dY, _ = synth.layer_inputs(5, M, K, N, kind="ternary")
    per = tp_layer(api, "2d", 4, 1, M, K, N, X, W, dY, None, "bf16", flags=FUSED | STAGED)
    for r in range(4):
        i, j = divmod(r, q)
        fwd = {("x", i, t) for t in range(q)} | {("w", t, j) for t in range(q)}
        bwd = ({("dy", i, t) for t in range(q)} | {("w", j, t) for t in range(q)}
               | {("x", t, i) for t in range(q)} | {("dy", t, j) for t in range(q)})
        size = {"x": mb * kq * 2, "w": kq * nq * 2, "dy": mb * nq * 2}
        exp = lambda s: sum(size[k] for (k, a, b) in s if (a, b) != (i, j))
        assert per[r]["staged_fwd"] == exp(fwd), r
        assert per[r]["staged_bwd"] == exp(bwd), r
        # forward = SUMMA's received bytes: (q-1) X panels + (q-1) W panels
        assert per[r]["staged_fwd"] == (q - 1) * (size["x"] + size["w"])
