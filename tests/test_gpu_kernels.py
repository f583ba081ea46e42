"""Single-GPU parity of the library's kernels against the oracle / the shared generator.

Tolerances: bf16 output rel-Frobenius <= 1e-2 (north star),
fp32 output of bf16 operands <= 2e-5 (fp32 accumulation only), fp32 mode <= 1e-5;
exact-integer inputs and every index / copy / generator path: bit-exact.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import dense
from oracle.grid import build_grid
from oracle.shards import LayerSpec, extent as oextent

from tp_harness import TORCH_DT, rel_fro, to_dev, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("kind,scale", [("uniform", 0.0625), ("uniform", 0.37), ("ternary", 1.0)])
def test_fill_bit_exact_vs_synth(api, dtype, kind, scale):
    rows, cols, r0, c0, gcols = 37, 129, 5, 11, 200
    ref = synth.tensor(42, 17, 64, gcols, kind, scale, dtype, row0=r0, nrows=rows, col0=c0, ncols=cols)
    out = torch.empty(rows, cols + 3, device="cuda", dtype=TORCH_DT[dtype])
    api.tp_fill(out, dtype, rows, cols, cols + 3, 42, 17, kind, scale, r0, c0, gcols)
    torch.cuda.synchronize()
    got = out[:, :cols].float().cpu().numpy()
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("mode,p,d,kw", [
    ("1d", 8, 1, dict(split_1d=0)), ("1d", 4, 1, dict(split_1d=1)), ("2d", 4, 1, {}),
    ("2d", 9, 1, {}), ("2.5d", 8, 2, {}), ("2.5d", 8, 2, dict(flags=1)), ("3d", 8, 1, dict(parity_3d=1)),
    ("3d", 27, 1, {})])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_pack_unpack_bit_exact(api, mode, p, d, kw, dtype):
    og = build_grid(mode, p, d)
    unit = {"1d": p, "2d": og.q, "2.5d": og.q * og.d, "3d": og.q * og.q}[mode]
    M, K, N = 3 * unit, 8 * unit, 5 * unit
    spec = LayerSpec(M, K, N, split_1d="row" if kw.get("split_1d") == 1 else "col",
                     parity=kw.get("parity_3d", 0), w_depth_sharded=bool(kw.get("flags", 0) & 1))
    ds = api.desc(M, K, N, dtype, **kw)
    for t, shp in (("X", (M, K)), ("W", (K, N)), ("Y", (M, N))):
        G = torch.arange(np.prod(shp), device="cuda", dtype=torch.float32).reshape(shp)
        G = (G % 251).to(TORCH_DT[dtype])          # exact in bf16
        back = torch.full_like(G, -1)
        for r in range(p):
            g = api.tp_grid_init(mode, p, r, 0, d)
            e = api.tp_shard_extent(g, ds, t)
            sh = torch.empty(e[1], e[3], device="cuda", dtype=G.dtype)
            api.tp_pack(g, ds, t, G, sh)
            oe = oextent(og, spec, r, t)
            ref = G[oe.row0:oe.row0 + oe.rows, oe.col0:oe.col0 + oe.cols]
            torch.cuda.synchronize()
            assert torch.equal(sh, ref)
            api.tp_unpack(g, ds, t, sh, back)
            api.tp_grid_destroy(g)
        torch.cuda.synchronize()
        assert torch.equal(back, G)


_WS = {}


def _gemm_ws(api):
    if "ws" not in _WS:
        _WS["ws"] = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    return _WS["ws"]


def _gemm_case(api, ta, tb, M, N, K, in_dt, out_dt, seed, alpha=1.0, with_c=False, with_bias=False,
               kind="uniform", pad=0, split_k=True):
    A = synth.tensor(seed, 0, K if ta else M, M if ta else K, kind, 1.0, in_dt)
    B = synth.tensor(seed, 1, N if tb else K, K if tb else N, kind, 0.5, in_dt)
    Cm = synth.tensor(seed, 2, M, N, "uniform", 1.0, "fp32") if with_c else None
    bias = synth.tensor(seed, 3, 1, N, "uniform", 1.0, in_dt)[0] if with_bias else None
    lda = A.shape[1] + pad
    ldb = B.shape[1] + pad
    dA = torch.zeros(A.shape[0], lda, device="cuda", dtype=TORCH_DT[in_dt])
    dA[:, :A.shape[1]] = to_dev(A, in_dt)
    dB = torch.zeros(B.shape[0], ldb, device="cuda", dtype=TORCH_DT[in_dt])
    dB[:, :B.shape[1]] = to_dev(B, in_dt)
    dC = to_dev(Cm, "fp32") if with_c else None
    db = to_dev(bias[None, :], in_dt)[0].contiguous() if with_bias else None
    D = torch.full((M, N), float("nan"), device="cuda", dtype=TORCH_DT[out_dt])
    api.tp_gemm(ta, tb, M, N, K, in_dt, dA, lda, dB, ldb, dC, N, D, N, out_dt, alpha, db,
                ws=_gemm_ws(api) if split_k else None)
    torch.cuda.synchronize()
    opA = A.T if ta else A
    opB = B.T if tb else B
    ref = dense.matmul(opA, opB)
    if with_c:
        ref = ref + Cm
    ref = alpha * ref
    if with_bias:
        ref = ref + bias[None, :]
    return to_np(D), ref


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (200, 136, 72), (384, 520, 256), (16, 64, 32),
                                   (1000, 1304, 328)])
def test_gemm_bf16_vs_oracle(api, ta, tb, M, N, K):
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "fp32", seed=M + N + K)
    assert rel_fro(got, ref) <= 2e-5
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "bf16", seed=M + N + K)
    assert rel_fro(got, ref) <= 1e-2 and np.isfinite(got).all()


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_bf16_exact_integer_bit_equal(api, ta, tb):
    """Ternary operands, K <= 256: exact products and sums, bf16-exact outputs (|y| <= 256)."""
    for (M, N, K) in [(128, 256, 256), (72, 40, 200), (304, 520, 136)]:
        got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "bf16", seed=7, kind="ternary")
        assert np.array_equal(got, ref)
        got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "fp32", seed=8, kind="ternary")
        assert np.array_equal(got, ref)


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(512, 4096, 4096), (304, 600, 1024), (264, 520, 2048)])
@pytest.mark.parametrize("split_k", [True, False])
def test_gemm_pair_kernel_split_k(api, ta, tb, M, N, K, split_k):
    """CTA-pair kernel with (and without) split-K: few 256x256 tiles, long K (C2 shapes)."""
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "fp32", seed=13, split_k=split_k)
    assert rel_fro(got, ref) <= 2e-5
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "bf16", seed=13, alpha=0.5, with_c=True,
                          with_bias=True, split_k=split_k)
    assert rel_fro(got, ref) <= 1e-2


def test_gemm_split_k_is_deterministic(api):
    A = to_dev(synth.tensor(1, 0, 512, 4096), "bf16")
    B = to_dev(synth.tensor(1, 1, 4096, 4096, scale=0.03), "bf16")
    outs = []
    for _ in range(3):
        D = torch.empty(512, 4096, device="cuda", dtype=torch.float32)
        api.tp_gemm(0, 0, 512, 4096, 4096, "bf16", A, 4096, B, 4096, None, 4096, D, 4096, "fp32",
                    ws=_gemm_ws(api))
        outs.append(D)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("env", [
    {"TP_GEMM_KERNEL": "1"},                                   # 1-CTA kernel everywhere
    {"TP_GEMM_KERNEL": "2"},                                   # CTA-pair kernel (M > 128)
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_MC": "2"},                # + A multicast over 2 pairs
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_MC": "3"},                # + B multicast over 2 pairs
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_MC": "4"},                # 2x2 pairs, A and B multicast
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_MC": "4", "TP_GEMM_BN": "128"},
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_MC": "5"},                # K-split pair cluster (DSMEM)
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_MC": "5", "TP_GEMM_BN": "128"},
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_BN": "128"},              # 256x128 pair tiles
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_BN": "256", "TP_GEMM_SPLITK": "0"},
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_BN": "256", "TP_GEMM_EPI_WARPS": "8"},  # 8 epilogue warps
    {"TP_GEMM_KERNEL": "2", "TP_GEMM_WIDE": "1"},              # 512x256 pair tiles wherever legal
    {"TP_GEMM_NARROW": "0"},                                   # ragged last n-tile at full width
], ids=lambda e: "-".join(f"{k[8:]}{v}" for k, v in e.items()))
def test_gemm_kernel_variants_forced(api, env):
    """Every kernel variant the dispatcher can pick, forced for every shape of the GEMM parity
    tests; run in a child process (the choice is read once per process)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, **env)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "tests/test_gpu_kernels.py",
                        "-k", "(bf16_vs_oracle or exact_integer or wide_tile or epilogue or pair_kernel or short_k"
                              " or deterministic or wide_pair or narrow) and not variants_forced"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 0), (0, 1)])
@pytest.mark.parametrize("M,N,K", [(2560, 2048, 64), (2600, 2056, 120)])
def test_gemm_short_k_eight_epilogue_warps(api, ta, tb, M, N, K):
    """<= 2 k-blocks per 256x256 tile and enough tiles: the dispatcher's 8-epilogue-warp pair
    kernel (ragged tails included)."""
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "fp32", seed=17)
    assert rel_fro(got, ref) <= 2e-5
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "bf16", seed=17, alpha=0.5, with_c=True,
                          with_bias=True)
    assert rel_fro(got, ref) <= 1e-2


def test_gemm_bf16_wide_tile_path(api):
    """Enough 128x256 tiles to take the BN=256 persistent path (> #SMs tiles), multi-tile per CTA."""
    for ta, tb in [(0, 0), (0, 1), (1, 0)]:
        got, ref = _gemm_case(api, ta, tb, 2048, 4096, 512, "bf16", "fp32", seed=3)
        assert rel_fro(got, ref) <= 2e-5


@pytest.mark.parametrize("ta,tb", [(0, 0), (1, 1)])
def test_gemm_epilogue_alpha_c_bias_and_padding(api, ta, tb):
    got, ref = _gemm_case(api, ta, tb, 264, 200, 136, "bf16", "fp32", seed=5, alpha=0.75,
                          with_c=True, with_bias=True, pad=8)
    assert rel_fro(got, ref) <= 2e-5
    got, ref = _gemm_case(api, ta, tb, 264, 200, 136, "bf16", "bf16", seed=5, alpha=-1.5,
                          with_c=True, with_bias=True)
    assert rel_fro(got, ref) <= 1e-2


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(16, 64, 64), (67, 45, 33), (130, 70, 260)])
def test_gemm_fp32_mode_vs_oracle(api, ta, tb, M, N, K):
    got, ref = _gemm_case(api, ta, tb, M, N, K, "fp32", "fp32", seed=11, alpha=0.5, with_c=True,
                          with_bias=True)
    assert rel_fro(got, ref) <= 1e-5


def test_gemm_degenerate_shapes(api):
    # K == 0: D = alpha * C + bias ; M == 0 / N == 0: nothing
    got, ref = _gemm_case(api, 0, 0, 32, 48, 0, "bf16", "fp32", seed=1, alpha=2.0, with_c=True,
                          with_bias=True)
    assert np.allclose(got, ref, rtol=1e-6, atol=1e-6)
    D = torch.zeros(4, 4, device="cuda")
    api.tp_gemm(0, 0, 0, 4, 8, "bf16", None, 8, None, 8, None, 4, D, 4, "fp32")
    with pytest.raises(api.TPError) as e:     # TMA stride rule: lda must be a multiple of 8
        A = torch.zeros(8, 12, device="cuda", dtype=torch.bfloat16)
        api.tp_gemm(0, 0, 8, 8, 12, "bf16", A, 12, A, 8, None, 8, D, 8, "fp32")
    assert e.value.status == 3


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_colsum_vs_oracle(api, dtype):
    for rows, cols in [(1000, 136), (7, 3), (4096, 520)]:
        Y = synth.tensor(9, 2, rows, cols, "uniform", 1.0, dtype)
        out = torch.empty(cols, device="cuda", dtype=TORCH_DT[dtype])
        api.tp_colsum(to_dev(Y, dtype), rows, cols, cols, dtype, out)
        torch.cuda.synchronize()
        ref = np.asarray(Y, np.float64).sum(axis=0)
        assert rel_fro(to_np(out), ref) <= (1e-2 if dtype == "bf16" else 1e-5)


def test_instrumentation_counts_launches_and_times_gemms(api):
    api.tp_prof_reset()
    api.tp_prof_enable(True)
    n0 = api.tp_launch_count()
    _gemm_case(api, 0, 0, 256, 256, 256, "bf16", "fp32", seed=2)
    api.tp_prof_enable(False)
    ms, n, fl = api.tp_prof_read(0)
    assert n == 1 and ms > 0 and fl == 2.0 * 256 ** 3
    assert api.tp_launch_count() - n0 >= 1
    api.tp_prof_reset()


@pytest.mark.parametrize("M,N,K,ldd", [(197, 197, 64, 200), (130, 130, 64, 136), (300, 197, 128, 256),
                                       (64, 20, 64, 24), (512, 516, 64, 520)])
@pytest.mark.parametrize("out", ["fp32", "bf16"])
def test_gemm_writes_only_inside_d(api, M, N, K, ldd, out):
    """D rows padded to ldd > N: the columns [N, ldd) of every row stay untouched (a TMA store of
    a ragged row's last 16-byte granule would zero them - the score padding of the ragged
    attention backward depended on it), and the M x N block is right."""
    A = torch.from_numpy(synth.tensor(5, 0, M, K)).cuda().to(torch.bfloat16)
    B = torch.from_numpy(synth.tensor(5, 1, K, N)).cuda().to(torch.bfloat16)
    dt = torch.float32 if out == "fp32" else torch.bfloat16
    D = torch.full((M, ldd), float("-inf"), device="cuda", dtype=dt)
    ws = torch.empty(api.tp_gemm_ws_bytes(), device="cuda", dtype=torch.uint8)
    ldb = (N + 7) // 8 * 8          # B's row stride must be a multiple of 8 elements (TMA)
    Bp = torch.zeros(K, ldb, device="cuda", dtype=torch.bfloat16)
    Bp[:, :N] = B
    api.tp_gemm(0, 0, M, N, K, "bf16", A, K, Bp, ldb, None, 0, D, ldd, out, 1.0, None, None, ws)
    torch.cuda.synchronize()
    assert bool(torch.isinf(D[:, N:]).all()), "GEMM wrote outside D[:, :N]"
    ref = dense.matmul(to_np(A), to_np(B))
    assert rel_fro(to_np(D[:, :N]), ref) <= (2e-5 if out == "fp32" else 1e-2)


@pytest.mark.parametrize("M,K,N,ta", [(192, 65536, 576, 1), (256, 32768, 384, 0), (136, 16384, 200, 1)])
def test_gemm_few_tiles_long_k(api, M, K, N, ta):
    """Few output tiles, long K (C4's QKV dW shape class): dispatched to the split-K pair
    kernel; fp32 out against the oracle."""
    got, ref = _gemm_case(api, ta, 0, M, N, K, "bf16", "fp32", seed=M + K, split_k=True)
    assert rel_fro(got, ref) <= 2e-5


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_wide_pair_tiles(api, ta, tb):
    """Shapes the dispatcher sends to the 512 x 256 pair-tile kernel (>= 74 tiles, K >= 4096),
    incl. ragged M / N tails: fp32 out exact to accumulation order, bf16 with alpha, C and bias."""
    for (M, N, K) in [(4096, 4608, 4096), (4000, 4616, 4160)]:
        got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "fp32", seed=29)
        assert rel_fro(got, ref) <= 2e-5
        got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "bf16", seed=29, alpha=0.5, with_c=True,
                              with_bias=True)
        assert rel_fro(got, ref) <= 1e-2


@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(10240, 384, 256), (9000, 264, 200), (10000, 640, 136)])
def test_gemm_narrow_last_tile(api, ta, tb, M, N, K):
    """256 x 256 pair tiles whose last n-tile holds <= 128 columns (C4's N = 384 products): that
    tile runs as an N = 128 pair MMA on half the B box (TP_GEMM_NARROW). Ragged M and a ragged
    narrow tail included; fp32 out exact to accumulation order, bf16 with alpha, C and bias."""
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "fp32", seed=31)
    assert rel_fro(got, ref) <= 2e-5
    got, ref = _gemm_case(api, ta, tb, M, N, K, "bf16", "bf16", seed=31, alpha=0.5, with_c=True,
                          with_bias=True)
    assert rel_fro(got, ref) <= 1e-2 and np.isfinite(got).all()


@pytest.mark.parametrize("sched", [1, 0])
@pytest.mark.parametrize("M,K,N", [(256, 3072, 3072), (200, 2056, 3000), (65536, 384, 256),
                                   (50000, 392, 264)])
def test_grouped_backward_unit_schedule(api, sched, M, K, N):
    """A layer backward whose grouped launch mixes units of unequal length: long-K dX tiles
    (K = N) next to many short dW tiles (K = M) (C2-like), or a long-K dW split into split-K
    units next to many short dX tiles (C4-like, M >> K, N). More units than pair clusters: the
    longest-first unit schedule (TP_GEMM_SCHED=1) assigns the C2-like launches (split-K launches
    keep round robin); round robin (0) for comparison. Both must match the oracle (dX, dW: every
    tile, ragged tails included)."""
    from tp_harness import gather, oracle_layer, spec_of, tp_layer
    old = api.tp_knob_get("TP_GEMM_SCHED")
    api.tp_knob_set("TP_GEMM_SCHED", sched)
    try:
        X, W, dY, _ = synth.layer_inputs(23, M, K, N)
        per = tp_layer(api, "1d", 1, 1, M, K, N, X, W, dY)
    finally:
        api.tp_knob_set("TP_GEMM_SCHED", old)
    spec = spec_of(M, K, N)
    ref = oracle_layer("1d", 1, 1, spec, X, W, dY)
    for (key, t), r in zip((("Y", "Y"), ("dX", "X"), ("dW", "W")), ref):
        assert rel_fro(gather("1d", 1, 1, spec, per, key, t), r) <= 1e-2, key
