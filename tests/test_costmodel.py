"""The library's analytic cost model (tp_cost_model, NEXT-4's comm-volume/scaling CLI) against
the oracle's closed forms, which are themselves pinned to the paper's Table and to
the simulated-collective ledger (tests/test_oracle_pins.py). Host only: runs without a GPU."""
from fractions import Fraction

import pytest

from oracle import closed_forms as cf

api = pytest.importorskip("paper_2110_14883_b200.api")

GRIDS = [("1d", 1, 0, 1), ("1d", 2, 0, 1), ("1d", 4, 0, 1), ("1d", 8, 0, 1), ("1d", 6, 0, 1),
         ("2d", 1, 1, 1), ("2d", 4, 2, 1), ("2d", 9, 3, 1), ("2d", 16, 4, 1),
         ("2.5d", 4, 2, 1), ("2.5d", 8, 2, 2), ("2.5d", 18, 3, 2), ("2.5d", 32, 2, 8),
         ("3d", 1, 1, 1), ("3d", 8, 2, 1), ("3d", 27, 3, 1)]
SHAPES = [(144, 96, 72), (512, 4096, 4096), (16384, 8192, 24576), (72, 216, 144)]


def _ok(mode, p, q, d, M, K, N, split):
    if mode == "1d":
        return (N if split == 0 else K) % p == 0
    if mode == "2d":
        return M % q == 0 and K % q == 0 and N % q == 0
    if mode == "2.5d":
        return M % (d * q) == 0 and K % q == 0 and N % q == 0
    return M % (q * q) == 0 and K % (q * q) == 0 and N % q == 0


@pytest.mark.parametrize("grid", GRIDS, ids=lambda g: f"{g[0]}-p{g[1]}-d{g[3]}")
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "x".join(map(str, s)))
@pytest.mark.parametrize("split", [0, 1])
def test_volumes_match_oracle(grid, shape, split):
    mode, p, q, d = grid
    M, K, N = shape
    if mode != "1d" and split:
        pytest.skip("split applies to 1D only")
    if not _ok(mode, p, q, d, M, K, N, split):
        pytest.skip("indivisible")
    c = api.tp_cost_model(mode, p, api.desc(M, K, N, "bf16", split_1d=split), q=q, depth=d)
    Sx, Sw, Sy = M * K, K * N, M * N
    if mode == "1d":
        paper = cf.paper_comm_volume("1d", Sy if split else Sx, Sw, p=p)
    elif mode == "2d":
        paper = cf.paper_comm_volume("2d", Sx, Sw, j=q)
    elif mode == "2.5d":
        paper = cf.paper_comm_volume("2.5d", Sx, Sw, k=q, d=d)
    else:
        paper = cf.paper_comm_volume("3d", Sx, Sw, Sy, l=q)
    counted = cf.counted_volume(mode, M, K, N, p=p, q=q, d=d, split_1d="row" if split else "col")
    assert c["paper_elems"] == pytest.approx(float(Fraction(paper)), rel=1e-12)
    assert c["counted_elems"] == pytest.approx(float(counted), rel=1e-12)
    assert c["link_bytes"] == pytest.approx(counted / p * 2, rel=1e-12)
    assert c["flops"] == pytest.approx(6.0 * M * K * N / p, rel=1e-12)
    mem = cf.memory_per_rank(mode, M, K, N, p, q=q, d=d, split_1d="row" if split else "col")
    assert (c["mem_x"], c["mem_w"], c["mem_y"]) == (mem["X"], mem["W"], mem["Y"])


def test_depth_sharded_weight_memory():
    c = api.tp_cost_model("2.5d", 8, api.desc(512, 4096, 4096, "bf16", flags=1), q=2, depth=2)
    assert c["mem_w"] == cf.memory_per_rank("2.5d", 512, 4096, 4096, 8, q=2, d=2,
                                            w_depth_sharded=True)["W"]


def test_roofline_times_and_survey_table():
    """SURVEY 8(d) roofline rows for C2 (two square layers, M=512, h=4096, F = 1663.3 TF/s,
    900 GB/s): per-GPU NVLink MB and the bound / max % of peak. F is pinned to SURVEY's value,
    not read from MEASURED_PEAKS.json (driver-written, changes between rounds)."""
    from paper_2110_14883_b200 import costmodel
    rows = {(r["grid"], r["gpus"]): r for p in (4, 8)
            for r in costmodel.model("c2", p, peak_tflops=1663.3)}
    assert rows[("1d", 4)]["link_mb_per_gpu"] == 12.6
    assert rows[("2d", 4)]["link_mb_per_gpu"] == 56.6 and rows[("2d", 4)]["bound"] == "link"
    assert rows[("2.5d(d=2)", 8)]["link_mb_per_gpu"] == 70.3
    assert rows[("3d", 8)]["link_mb_per_gpu"] == 21.0
    assert rows[("3d", 8)]["max_pct_of_peak"] == 33.2
    assert rows[("1d", 8)]["max_pct_of_peak"] == 47.5


def test_errors():
    with pytest.raises(api.TPError):
        api.tp_cost_model("2d", 8, api.desc(16, 16, 16))  # 8 is not a square
    with pytest.raises(api.TPError):
        api.tp_cost_model("3d", 8, api.desc(6, 16, 16))  # M not divisible by l^2


@pytest.mark.parametrize("q", [2, 3, 4])
def test_cannon_volume_matches_oracle_ledger(q):
    """Cannon's volume (forward: SUMMA's plus the skew; backward: moving accumulators, reading N7)
    equals the message count of the oracle's Cannon programs (oracle/cannon.py)."""
    import numpy as np
    from oracle import cannon
    from oracle.fabric import Fabric
    from oracle.grid import build_grid
    from oracle.shards import LayerSpec, shard
    M, K, N = 6 * q, 4 * q, 2 * q
    grid = build_grid("2d", q * q)
    spec = LayerSpec(M, K, N)
    fab = Fabric()
    X, W = np.ones((M, K)), np.ones((K, N))
    cannon.cannon_fwd(grid, shard(grid, spec, X, "X"), shard(grid, spec, W, "W"), fab=fab)
    cannon.cannon_bwd(grid, shard(grid, spec, np.ones((M, N)), "Y"), shard(grid, spec, X, "X"),
                      shard(grid, spec, W, "W"), fab=fab)
    c0 = api.tp_cost_model("2d", q * q, api.desc(M, K, N), q=q)
    c1 = api.tp_cost_model("2d", q * q, api.desc(M, K, N, flags=0x10), q=q)
    summa = cf.counted_volume("2d", M, K, N, q=q, part="fwd+bwd")
    assert c0["counted_elems"] == pytest.approx(summa)
    assert c1["counted_elems"] == pytest.approx(fab.ledger.total())


def test_solomonik_volume_equals_oracle():
    """TP_FLAG_SOLOMONIK (reading N5): the cost model's counted volume and shard sizes equal
    oracle/solomonik.py's closed form and its layout."""
    from oracle import solomonik as so
    from oracle.grid import build_grid
    from oracle.shards import LayerSpec
    for (q, d) in [(2, 2), (4, 2), (2, 1)]:
        M, K, N = 64 * q, 32 * q, 48 * q
        c = api.tp_cost_model("2.5d", d * q * q, api.desc(M, K, N, "bf16", flags=api.TP_FLAG_SOLOMONIK),
                              q=q, depth=d)
        grid, spec = build_grid("2.5d", d * q * q, d), LayerSpec(M, K, N)
        cf = so.closed_form_volume(grid, spec)
        assert c["counted_elems"] == cf["fwd"] + cf["bwd"]
        e = so.extent(grid, spec, 0, "W")
        assert c["mem_w"] == e.rows * e.cols


def test_solomonik_extents_match_oracle():
    from oracle import solomonik as so
    from oracle.grid import build_grid
    from oracle.shards import LayerSpec
    q, d = 2, 2
    M, K, N = 96, 64, 80
    grid, spec = build_grid("2.5d", 8, 2), LayerSpec(M, K, N)
    ds = api.desc(M, K, N, "bf16", flags=api.TP_FLAG_SOLOMONIK)
    for r in range(8):
        g = api.tp_grid_init("2.5d", 8, r, 0, 2, 0, api.TP_TRANSPORT_NONE)
        try:
            for t in ("X", "W", "Y", "B"):
                e = so.extent(grid, spec, r, t)
                assert api.tp_shard_extent(g, ds, t) == (e.row0, e.rows, e.col0, e.cols)
        finally:
            api.tp_grid_destroy(g)
    with pytest.raises(api.TPError):   # q = 2 is not divisible by d = 4 ... (p = 16, q = 2, d = 4)
        api.tp_cost_model("2.5d", 16, ds, q=2, depth=4)


def test_exposed_comm_term():
    """The exposed-communication estimate: 0 on one GPU; never more than the whole transfer
    time; the 3D row-block pipeline leaves less exposed than 2D SUMMA at q=2 for C3-HEAD (what the
    pipelining is for); more link bandwidth never exposes more."""
    from paper_2110_14883_b200 import api
    M = h = 16384
    for mode, p in (("1d", 1), ("2d", 1), ("3d", 1)):
        c = api.tp_cost_model(mode, p, api.desc(M, h, h), peak_tflops=1500, link_gbs=900)
        assert c["t_exposed_us"] == 0
    for mode, p, flags in (("1d", 8, 0), ("2d", 4, 0), ("2.5d", 8, 0), ("2.5d", 8, 1), ("3d", 8, 0)):
        d = 2 if mode == "2.5d" else 1
        for par in (0, 1):
            ds = api.desc(M, h, h, split_1d=par, parity_3d=par, flags=flags)
            c = api.tp_cost_model(mode, p, ds, depth=d, peak_tflops=1500, link_gbs=900)
            assert 0 <= c["t_exposed_us"] <= c["t_link_us"] * 1.0000001 + 1e-9, (mode, par)
            c2 = api.tp_cost_model(mode, p, ds, depth=d, peak_tflops=1500, link_gbs=1800)
            assert c2["t_exposed_us"] <= c["t_exposed_us"] + 1e-9
    e3 = api.tp_cost_model("3d", 8, api.desc(M, h, h), peak_tflops=1500, link_gbs=900)
    e2 = api.tp_cost_model("2d", 4, api.desc(M, h, h), peak_tflops=1500, link_gbs=900)
    assert e3["t_exposed_us"] < e2["t_exposed_us"]


def test_fused_peer_bytes():
    """The fused owner-computes path's NVLink bytes per rank: panels read straight from peers
    are re-read once per 256-wide output tile (C3-HEAD 2D: ~32x SUMMA's volume); staged
    (TP_FLAG_PEER_STAGED) each remote shard crosses once - for 2D exactly the collective
    schedule's received bytes."""
    from paper_2110_14883_b200 import api
    M = h = 16384
    for par in (0, 1):
        c = api.tp_cost_model("2d", 4, api.desc(M, h, h, split_1d=par, parity_3d=par))
        assert c["fused_staged_bytes"] == pytest.approx(c["link_bytes"], rel=1e-12)
        assert c["fused_direct_bytes"] > 20 * c["fused_staged_bytes"]
        c3 = api.tp_cost_model("3d", 8, api.desc(M, h, h, split_1d=par, parity_3d=par))
        assert c3["fused_direct_bytes"] > 10 * c3["fused_staged_bytes"] > 0
    c1 = api.tp_cost_model("1d", 8, api.desc(M, h, h))
    assert c1["fused_direct_bytes"] == 0 and c1["fused_staged_bytes"] == 0
