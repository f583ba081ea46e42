"""GPU parity of the tensor-parallel LayerNorm (tp_layernorm_fwd / _bwd)
against the oracle (oracle/layernorm.py: dense definition, pinned in
tests/test_oracle_layernorm.py). Ranks are in-process threads on cuda:0 (LOCAL transport)."""
import numpy as np
import pytest
import torch

import synth
from oracle import layernorm as ln
from oracle.grid import build_grid
from oracle.shards import extent as oextent

from tp_harness import TORCH_DT, gather, rel_fro, run_ranks, spec_of, to_dev, to_np

pytestmark = pytest.mark.gpu

LAYOUTS = [("1d", 1, 1, 0, 0, "X"), ("1d", 4, 1, 0, 0, "Y"), ("1d", 4, 1, 1, 0, "X"),
           ("1d", 4, 1, 1, 0, "Y"), ("2d", 4, 1, 0, 0, "X"), ("2d", 9, 1, 0, 0, "Y"),
           ("2.5d", 8, 2, 0, 0, "X"), ("2.5d", 8, 2, 0, 0, "Y"),
           ("3d", 8, 1, 0, 0, "X"), ("3d", 8, 1, 0, 1, "X"), ("3d", 8, 1, 0, 0, "Y"),
           ("3d", 8, 1, 0, 1, "Y")]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def _inputs(seed, M, H, dtype):
    q = "bf16" if dtype == "bf16" else "fp32"
    X = synth.tensor(seed, 0, M, H, dtype=q).astype(np.float64)
    g = synth.tensor(seed, 1, 1, H, dtype=q)[0].astype(np.float64) * 0.5 + 1.0
    b = synth.tensor(seed, 2, 1, H, dtype=q)[0].astype(np.float64) * 0.1
    dY = synth.tensor(seed, 3, M, H, dtype=q).astype(np.float64)
    # gamma / beta are used as stored: quantise the affine transform's result the same way
    cast = (lambda a: torch.tensor(a).to(torch.bfloat16).double().numpy()) if dtype == "bf16" else (lambda a: a)
    return X, cast(g), cast(b), dY


def run_ln(api, mode, p, d, M, K, N, split, par, tensor, dtype, X, g, b, dY, eps=1e-5):
    transport = api.TP_TRANSPORT_LOCAL if p > 1 else api.TP_TRANSPORT_NONE
    uid = api.tp_get_unique_id(transport)
    gX, gdY = to_dev(X, dtype), to_dev(dY, dtype)
    torch.cuda.synchronize()

    def rank_fn(r):
        grid = api.tp_grid_init(mode, p, r, 0, d, 0, transport, uid)
        s = torch.cuda.Stream()
        try:
            with torch.cuda.stream(s):
                ds = api.desc(M, K, N, dtype, split, par)
                r0, rows, c0, cols = api.tp_shard_extent(grid, ds, tensor)
                mk = lambda: torch.empty(rows, cols, device="cuda", dtype=TORCH_DT[dtype])
                x, y, dy, dx = mk(), mk(), mk(), mk()
                api.tp_pack(grid, ds, tensor, gX, x)
                api.tp_pack(grid, ds, tensor, gdY, dy)
                gam = to_dev(g[None, c0:c0 + cols], dtype)[0].contiguous()
                bet = to_dev(b[None, c0:c0 + cols], dtype)[0].contiguous()
                stats = torch.empty(rows, 2, device="cuda", dtype=torch.float32)
                ws = torch.empty(max(api.tp_layernorm_ws_size(grid, ds, tensor), 1), device="cuda",
                                 dtype=torch.uint8)
                api.tp_layernorm_fwd(grid, ds, tensor, eps, x, gam, bet, y, stats, ws)
                dg = torch.empty(cols, device="cuda", dtype=TORCH_DT[dtype])
                db = torch.empty(cols, device="cuda", dtype=TORCH_DT[dtype])
                api.tp_layernorm_bwd(grid, ds, tensor, dy, x, gam, stats, dx, dg, db, ws)
            s.synchronize()
            return {"Y": to_np(y), "dX": to_np(dx), "dg": to_np(dg), "db": to_np(db),
                    "stats": stats.double().cpu().numpy(), "ext": (r0, rows, c0, cols)}
        finally:
            s.synchronize()
            api.tp_grid_destroy(grid)

    return run_ranks(p, rank_fn)


@pytest.mark.parametrize("lay", LAYOUTS, ids=lambda l: "-".join(map(str, l)))
@pytest.mark.parametrize("dtype", ["fp32", "bf16"])
def test_layernorm_vs_oracle(api, lay, dtype):
    mode, p, d, split, par, tensor = lay
    M, K, N = 144, 72, 144
    H = K if tensor == "X" else N
    X, g, b, dY = _inputs(7, M, H, dtype)
    eps = 1e-5
    per = run_ln(api, mode, p, d, M, K, N, split, par, tensor, dtype, X, g, b, dY, eps)
    Yd, mu, rstd = ln.ln_fwd(X, g, b, eps)
    dXd, dgd, dbd = ln.ln_bwd(dY, X, g, mu, rstd)
    spec = spec_of(M, K, N, split, par)
    tol = 1e-5 if dtype == "fp32" else 1e-2
    assert rel_fro(gather(mode, p, d, spec, per, "Y", tensor), Yd) <= tol
    assert rel_fro(gather(mode, p, d, spec, per, "dX", tensor), dXd) <= tol
    for r in range(p):
        r0, rows, c0, cols = per[r]["ext"]
        assert rel_fro(per[r]["dg"], dgd[c0:c0 + cols]) <= tol
        assert rel_fro(per[r]["db"], dbd[c0:c0 + cols]) <= tol
        # saved statistics are the rows' exact mean and 1/sqrt(var + eps) (fp32)
        assert np.allclose(per[r]["stats"][:, 0], mu[r0:r0 + rows], rtol=1e-5, atol=1e-6)
        assert np.allclose(per[r]["stats"][:, 1], rstd[r0:r0 + rows], rtol=1e-4)


def test_layernorm_replicas_bit_equal(api):
    """Every replica of a block (and of dgamma/dbeta) is bit-identical: the fp32 reductions are
    deterministic all-reduces and the column sums use fixed row slabs."""
    M, K, N = 256, 128, 256
    X, g, b, dY = _inputs(3, M, K, "bf16")
    per = run_ln(api, "3d", 8, 1, M, K, N, 0, 0, "X", "bf16", X, g, b, dY)
    grid = build_grid("3d", 8)
    spec = spec_of(M, K, N)
    seen = {}
    for r in range(8):
        e = oextent(grid, spec, r, "X")
        key = (e.col0, e.cols)
        if key in seen:
            assert np.array_equal(per[r]["dg"], per[seen[key]]["dg"])
            assert np.array_equal(per[r]["db"], per[seen[key]]["db"])
        seen.setdefault(key, r)


def test_layernorm_fullsize_bf16(api):
    """A transformer-sized activation (C2/C5 hidden sizes): 2D q=2 over M=2048, H=8192."""
    M, K, N = 2048, 8192, 8192
    X, g, b, dY = _inputs(9, M, K, "bf16")
    per = run_ln(api, "2d", 4, 1, M, K, N, 0, 0, "X", "bf16", X, g, b, dY)
    Yd, mu, rstd = ln.ln_fwd(X, g, b, 1e-5)
    dXd, dgd, dbd = ln.ln_bwd(dY, X, g, mu, rstd)
    spec = spec_of(M, K, N)
    assert rel_fro(gather("2d", 4, 1, spec, per, "Y", "X"), Yd) <= 1e-2
    assert rel_fro(gather("2d", 4, 1, spec, per, "dX", "X"), dXd) <= 1e-2
