"""GPU parity of the multi-head attention core in the TP layouts (tp_attention_fwd / _bwd,
SURVEY 8(f) NEXT-2) against the oracle (oracle/mha.py, pinned in tests/test_oracle_mha.py).
The QKV output block of each rank is attended locally; the result is the X block of the output
projection. In-process ranks on cuda:0."""
import numpy as np
import pytest
import torch

import synth
from oracle import mha
from oracle.grid import build_grid
from oracle.shards import gather_full

from tp_harness import TORCH_DT, rel_fro, run_ranks, spec_of, to_dev, to_np

pytestmark = pytest.mark.gpu

# (mode, p, d, qkv split/parity, proj split/parity)
LAYOUTS = [("1d", 1, 1, 0, 1), ("1d", 4, 1, 0, 1), ("2d", 4, 1, 0, 0), ("2.5d", 8, 2, 0, 0),
           ("3d", 8, 1, 0, 1)]


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


def run_attn(api, mode, p, d, M, h, seq, heads, dtype, qkv, dout, sq, sp, fused_bwd=False):
    transport = api.TP_TRANSPORT_LOCAL if p > 1 else api.TP_TRANSPORT_NONE
    uid = api.tp_get_unique_id(transport)
    gq, gd = to_dev(qkv, dtype), to_dev(dout, dtype)
    torch.cuda.synchronize()

    def rank_fn(r):
        g = api.tp_grid_init(mode, p, r, 0, d, 0, transport, uid)
        st = torch.cuda.Stream()
        try:
            with torch.cuda.stream(st):
                dq = api.desc(M, h, 3 * h, dtype, split_1d=sq, parity_3d=sq)
                dp = api.desc(M, h, h, dtype, split_1d=sp, parity_3d=sp)
                eq = api.tp_shard_extent(g, dq, "Y")
                ep = api.tp_shard_extent(g, dp, "X")
                x = torch.empty(eq[1], eq[3], device="cuda", dtype=TORCH_DT[dtype])
                api.tp_pack(g, dq, "Y", gq, x)
                out = torch.empty(ep[1], ep[3], device="cuda", dtype=TORCH_DT[dtype])
                do = torch.empty_like(out)
                api.tp_pack(g, dp, "X", gd, do)
                ws = torch.empty(api.tp_attention_ws_size(g, dq, seq, heads), device="cuda",
                                 dtype=torch.uint8)
                hl = eq[3] // (3 * (h // heads))  # heads held by this rank
                lse = torch.empty(hl * eq[1], device="cuda", dtype=torch.float32) if fused_bwd else None
                api.tp_attention_fwd(g, dq, seq, heads, x, out, ws, lse=lse)
                dx = torch.empty_like(x)
                api.tp_attention_bwd(g, dq, seq, heads, x, do, dx, ws, out=out if fused_bwd else None,
                                     lse=lse)
            st.synchronize()
            return {"out": to_np(out), "dqkv": to_np(dx)}
        finally:
            st.synchronize()
            api.tp_grid_destroy(g)

    return run_ranks(p, rank_fn)


@pytest.mark.parametrize("lay", LAYOUTS, ids=lambda l: "-".join(map(str, l)))
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_attention_core_vs_oracle(api, lay, dtype):
    mode, p, d, sq, sp = lay
    seq, heads, dh = 128, 4, 64
    h = heads * dh
    M = seq * 8
    q = "bf16" if dtype == "bf16" else "fp32"
    qkv = synth.tensor(31, 0, M, 3 * h, dtype=q).astype(np.float64)
    dout = synth.tensor(31, 1, M, h, dtype=q).astype(np.float64)
    per = run_attn(api, mode, p, d, M, h, seq, heads, dtype, qkv, dout, sq, sp)
    grid = build_grid(mode, p, d)
    out = gather_full(grid, spec_of(M, h, h, sp, sp), {r: per[r]["out"] for r in range(p)}, "X")
    dqkv = gather_full(grid, spec_of(M, h, 3 * h, sq, sq), {r: per[r]["dqkv"] for r in range(p)}, "Y")
    tol = 1e-2 if dtype == "bf16" else 1e-5
    assert rel_fro(out, mha.mha_fwd(qkv, seq, heads)) <= tol
    assert rel_fro(dqkv, mha.mha_bwd(qkv, dout, seq, heads)) <= tol


@pytest.mark.parametrize("lay", LAYOUTS, ids=lambda l: "-".join(map(str, l)))
@pytest.mark.parametrize("seq,heads,dh", [(128, 4, 64), (256, 2, 128), (197, 6, 64), (300, 2, 128)])
def test_attention_fused_backward_vs_oracle(api, lay, seq, heads, dh):
    """bf16, d in {64, 128}: the forward writes the row log-sum-exp and the backward runs the
    fused kernel (flash_bwd.cu: P recomputed on chip, dQ accumulated across key tiles) - aligned
    and ragged sequences (197 = ViT-S/16, 300: a partial last tile of keys and of queries)."""
    mode, p, d, sq, sp = lay
    h = heads * dh
    nseq = 8
    M = seq * nseq
    qkv = synth.tensor(37, 0, M, 3 * h, dtype="bf16").astype(np.float64)
    dout = synth.tensor(37, 1, M, h, dtype="bf16").astype(np.float64)
    try:
        per = run_attn(api, mode, p, d, M, h, seq, heads, "bf16", qkv, dout, sq, sp, fused_bwd=True)
    except api.TPError as e:  # a layout whose blocks split a head (heads % column split)
        assert "head" in str(e)
        pytest.skip(str(e))
    grid = build_grid(mode, p, d)
    out = gather_full(grid, spec_of(M, h, h, sp, sp), {r: per[r]["out"] for r in range(p)}, "X")
    dqkv = gather_full(grid, spec_of(M, h, 3 * h, sq, sq), {r: per[r]["dqkv"] for r in range(p)}, "Y")
    assert rel_fro(out, mha.mha_fwd(qkv, seq, heads)) <= 1e-2
    ref = mha.mha_bwd(qkv, dout, seq, heads)
    assert rel_fro(dqkv, ref) <= 1e-2
    # each of dQ, dK, dV on its own (columns [q | k | v] per head)
    for c in range(3):
        cols = np.concatenate([np.arange(3 * dh * g + c * dh, 3 * dh * g + (c + 1) * dh) for g in range(heads)])
        assert rel_fro(dqkv[:, cols], ref[:, cols]) <= 1e-2, "qkv"[c]


def test_attention_rejects_split_heads_and_sequences(api):
    g = api.tp_grid_init("2d", 4, 0, 0, 1, 0, api.TP_TRANSPORT_NONE)
    with pytest.raises(api.TPError, match="sequence"):   # M/q = 96 rows, seq 128
        api.tp_attention_ws_size(g, api.desc(192, 256, 768), 128, 4)
    with pytest.raises(api.TPError, match="head"):       # 3h/q = 384 columns, head = 3 x 96
        api.tp_attention_ws_size(g, api.desc(256, 288, 864), 128, 3)
    api.tp_grid_destroy(g)
