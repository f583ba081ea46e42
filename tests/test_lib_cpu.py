"""Host-only checks of the C-ABI library (no GPU): it loads, exports every symbol the
header declares, and its grid / shard-extent / validation logic equals the oracle's
bit-exactly for every admissible grid up to p = 64 (SURVEY 4 "Grid tests")."""
import os
import re
import subprocess

import pytest

from oracle.grid import ConstraintViolation, build_grid
from oracle.shards import IndivisibleDim, LayerSpec, extent as oextent

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def api():
    from paper_2110_14883_b200 import build
    build.build()
    from paper_2110_14883_b200 import api
    return api


def header_functions():
    src = open(os.path.join(ROOT, "include", "tp_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(tp_\w+)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(api):
    from paper_2110_14883_b200 import _lib
    declared = header_functions()
    assert len(declared) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (tp_\w+)$", out, flags=re.M))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert set(_lib.EXPORTED) == set(declared)
    assert "sm_100a" in api.tp_version()


def test_sass_has_tcgen05_and_tma():
    """The product kernels are Blackwell-native: tcgen05 MMA (UTC*MMA), TMEM loads (LDTM)
    and TMA (UTMALDG) appear in the library's SASS."""
    from paper_2110_14883_b200 import _lib
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True,
                          check=True).stdout
    assert re.search(r"UTC\w*MMA", sass)
    assert "LDTM" in sass and "UTMALDG" in sass
    assert not re.search(r"\bHMMA\b", sass)   # no legacy mma.sync path


def admissible():
    out = []
    for p in range(1, 65):
        out.append(("1d", p, 1))
        for mode in ("2d", "3d"):
            try:
                build_grid(mode, p)
                out.append((mode, p, 1))
            except ConstraintViolation:
                pass
        for d in range(1, p + 1):
            try:
                build_grid("2.5d", p, d)
                out.append(("2.5d", p, d))
            except ConstraintViolation:
                pass
    return out


def test_grid_coords_and_groups_match_oracle(api):
    n = 0
    for mode, p, d in admissible():
        og = build_grid(mode, p, d)
        for r in range(p):
            g = api.tp_grid_init(mode, p, r, 0, d)
            try:
                c = api.tp_grid_coords(g)
                assert c[: len(og.dims)] == og.coords(r)
                assert api.tp_grid_dims(g) == og.dims
                for ax in range(len(og.dims)):
                    assert api.tp_grid_group(g, ax) == og.group(r, ax)
            finally:
                api.tp_grid_destroy(g)
            n += 1
    assert n > 500


@pytest.mark.parametrize("mode,p,d", [("2d", 8, 1), ("3d", 6, 1), ("2.5d", 8, 3), ("2.5d", 6, 2),
                                      ("2d", 2, 1), ("3d", 16, 1)])
def test_constraint_violation_status(api, mode, p, d):
    with pytest.raises(api.TPError) as e:
        api.tp_grid_init(mode, p, 0, 0, d)
    assert e.value.status == 1 and "needs" in str(e.value)


CASES = [
    ("1d", 4, 1, dict(split_1d=0)), ("1d", 4, 1, dict(split_1d=1)), ("1d", 8, 1, dict(split_1d=1)),
    ("2d", 4, 1, {}), ("2d", 9, 1, {}), ("2d", 16, 1, {}),
    ("2.5d", 4, 1, {}), ("2.5d", 8, 2, {}), ("2.5d", 8, 2, dict(flags=1)), ("2.5d", 18, 2, {}),
    ("3d", 8, 1, dict(parity_3d=0)), ("3d", 8, 1, dict(parity_3d=1)), ("3d", 27, 1, dict(parity_3d=1)),
]


@pytest.mark.parametrize("mode,p,d,kw", CASES)
def test_shard_extents_bit_exact_vs_oracle(api, mode, p, d, kw):
    og = build_grid(mode, p, d)
    unit = {"1d": p, "2d": og.q, "2.5d": og.q * og.d, "3d": og.q * og.q}[mode]
    M, K, N = 3 * unit, 2 * unit, 5 * unit
    spec = LayerSpec(M, K, N, split_1d="row" if kw.get("split_1d") == 1 else "col",
                     parity=kw.get("parity_3d", 0), w_depth_sharded=bool(kw.get("flags", 0) & 1))
    ds = api.desc(M, K, N, **kw)
    for r in range(p):
        g = api.tp_grid_init(mode, p, r, 0, d)
        try:
            for t in ("X", "W", "Y", "B"):
                e = oextent(og, spec, r, t)
                assert api.tp_shard_extent(g, ds, t) == (e.row0, e.rows, e.col0, e.cols)
        finally:
            api.tp_grid_destroy(g)


@pytest.mark.parametrize("mode,p,d,M,K,N,kw", [
    ("2d", 4, 1, 5, 4, 4, {}), ("3d", 8, 1, 8, 6, 4, {}), ("1d", 4, 1, 4, 4, 6, dict(split_1d=0)),
    ("2.5d", 8, 2, 8, 6, 4, dict(flags=1)), ("1d", 3, 1, 3, 4, 3, dict(split_1d=1))])
def test_indivisible_status_matches_oracle(api, mode, p, d, M, K, N, kw):
    og = build_grid(mode, p, d)
    spec = LayerSpec(M, K, N, split_1d="row" if kw.get("split_1d") == 1 else "col",
                     w_depth_sharded=bool(kw.get("flags", 0) & 1))
    with pytest.raises(IndivisibleDim):
        oextent(og, spec, 0, "X")
    g = api.tp_grid_init(mode, p, 0, 0, d)
    try:
        with pytest.raises(api.TPError) as e:
            api.tp_shard_extent(g, api.desc(M, K, N, **kw), "X")
        assert e.value.status == 2
    finally:
        api.tp_grid_destroy(g)


def test_workspace_sizes_cover_schedule_buffers(api):
    """ws / saved are at least the closed-form buffer footprints of SURVEY 8(c)-6."""
    M = K = N = 1024
    g = api.tp_grid_init("2d", 4, 0)
    ws, sv = api.tp_workspace_size(g, api.desc(M, K, N))
    api.tp_grid_destroy(g)
    q = 2
    # SUMMA double buffers: fwd 2 X + 2 W panels + fp32 accumulator; bwd two chains
    assert ws >= (2 * (M // q) * (K // q) + 2 * (K // q) * (N // q)) * 2 + (M // q) * (N // q) * 4
    assert sv == 0
    g = api.tp_grid_init("3d", 8, 0)
    ws, sv = api.tp_workspace_size(g, api.desc(M, K, N))
    api.tp_grid_destroy(g)
    assert sv >= ((M // 2) * (K // 2) + (K // 2) * (N // 2)) * 2     # gathered X and W kept
    g = api.tp_grid_init("1d", 1, 0)
    ws, sv = api.tp_workspace_size(g, api.desc(M, K, N))
    api.tp_grid_destroy(g)
    assert sv == 0


def test_compute_on_none_transport_needs_world_1(api):
    g = api.tp_grid_init("2d", 4, 0)
    try:
        with pytest.raises(api.TPError) as e:
            api.tp_linear_fwd(g, api.desc(4, 4, 4), 1, 1, None, 1, None, 1, stream=0,
                              ws_bytes=1 << 20)
        assert e.value.status == 4
    finally:
        api.tp_grid_destroy(g)


def test_rsa_and_layernorm_planning_errors():
    """Host-side checks of the NEXT-2/3 entry points (nothing is enqueued on error)."""
    from paper_2110_14883_b200 import api
    g2 = api.tp_grid_init("2d", 4, 0, 0, 1, 0, api.TP_TRANSPORT_NONE)
    with pytest.raises(api.TPError, match="1D"):
        api.tp_rsa_ws_size(g2, api.rsa_desc(64, 16, 1))
    with pytest.raises(api.TPError):
        api.tp_layernorm_ws_size(g2, api.desc(8, 8, 8), "W")  # LayerNorm of a weight
    api.tp_grid_destroy(g2)
    g3 = api.tp_grid_init("1d", 3, 0, 0, 1, 0, api.TP_TRANSPORT_NONE)
    with pytest.raises(api.TPError, match="divisible"):
        api.tp_rsa_ws_size(g3, api.rsa_desc(100, 16, 1))
    assert api.tp_rsa_ws_size(g3, api.rsa_desc(96, 16, 2)) > 2 * 32 * 96 * 4
    api.tp_grid_destroy(g3)


def test_tuning_knobs_registry(api):
    """Every dispatch / variant knob is in one registry: listed with its default and source,
    settable through the API, overridable by its TP_* environment variable (read once)."""
    import json
    import os
    import subprocess
    import sys
    ks = {k["name"]: k for k in api.tp_knobs()}
    for name in ("TP_PDL", "TP_GEMM_KERNEL", "TP_GEMM_WIDE", "TP_GEMM_RASTER", "TP_COMM_SMS",
                 "TP_FLASH", "TP_RSA_FUSED", "TP_GEMM_SPLITK", "TP_GEMM_SCHED", "TP_GEMM_SCHED_EPI",
                 "TP_GEMM_GROUP_LONGK", "TP_GEMM_L2PROMO"):
        assert name in ks and ks[name]["what"]
    assert ks["TP_GEMM_WIDE"]["default"] == -1 and ks["TP_PDL"]["default"] == 1
    # the measured defaults of session 3 (profiles/r02_c2_gemm.md)
    assert ks["TP_GEMM_SCHED"]["default"] == 1 and ks["TP_GEMM_SCHED_EPI"]["default"] == 800
    assert ks["TP_GEMM_GROUP_LONGK"]["default"] == 1 and ks["TP_GEMM_L2PROMO"]["default"] == 3
    old = api.tp_knob_get("TP_GEMM_RASTER")
    api.tp_knob_set("TP_GEMM_RASTER", 4)
    assert api.tp_knob_get("TP_GEMM_RASTER") == 4
    assert {k["name"]: k for k in api.tp_knobs()}["TP_GEMM_RASTER"]["source"] == "api"
    api.tp_knob_set("TP_GEMM_RASTER", old)
    with pytest.raises(api.TPError):
        api.tp_knob_set("TP_NO_SUCH_KNOB", 1)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import json; from paper_2110_14883_b200 import api; "
            "print(json.dumps({k['name']: k for k in api.tp_knobs()}['TP_GEMM_WIDE']))")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, TP_GEMM_WIDE="0"), timeout=120)
    k = json.loads(r.stdout.strip().splitlines()[-1])
    assert k["value"] == 0 and k["source"] == "env"
