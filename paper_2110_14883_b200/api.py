"""Python binding of the C ABI: the same names as include/tp_b200.h, argument marshalling only.

Tensors are torch tensors (their data_ptr() is passed) or raw integer device pointers;
None is NULL. `stream` defaults to torch's current CUDA stream. Every non-OK status
raises TPError carrying tp_last_error(). No compute happens here.
"""
from __future__ import annotations

import ctypes as C

from . import _lib as L
from ._lib import (TP_1D, TP_2D, TP_2P5D, TP_3D, TP_BF16, TP_FP32, TP_FLAG_SERIAL,  # noqa: F401
                   TP_FLAG_PEER_FUSED, TP_FLAG_GELU, TP_FLAG_CANNON, TP_FLAG_SOLOMONIK,
                   TP_FLAG_PEER_STAGED,
                   TP_FLAG_W25_DEPTH_SHARDED, TP_TENSOR_BIAS, TP_TENSOR_W, TP_TENSOR_X,
                   TP_TENSOR_Y, TP_TRANSPORT_LOCAL, TP_TRANSPORT_NCCL, TP_TRANSPORT_NONE,
                   tp_cost, tp_linear_desc, tp_rsa_desc)

lib = L.lib

MODES = {"1d": TP_1D, "2d": TP_2D, "2.5d": TP_2P5D, "3d": TP_3D}
DTYPES = {"bf16": TP_BF16, "fp32": TP_FP32}
TENSORS = {"X": TP_TENSOR_X, "W": TP_TENSOR_W, "Y": TP_TENSOR_Y, "B": TP_TENSOR_BIAS}


class TPError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib.tp_status_string(status).decode()
        detail = lib.tp_last_error().decode()
        super().__init__(f"{where}: {msg}: {detail}")


def _check(status: int, where: str):
    if status != L.TP_OK:
        raise TPError(status, where)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def desc(M, K, N, dtype="bf16", split_1d=0, parity_3d=0, flags=0, alpha=1.0) -> tp_linear_desc:
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    return tp_linear_desc(int(M), int(K), int(N), dt, int(split_1d), int(parity_3d), int(flags),
                          float(alpha))


def tp_version() -> str:
    return lib.tp_version().decode()


def tp_get_unique_id(transport: int) -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib.tp_get_unique_id(transport, buf), "tp_get_unique_id")
    return buf.raw


def share_unique_id(transport: int, src: int = 0) -> bytes:
    """Rank `src` creates the 128-byte id, torch.distributed broadcasts it (rendezvous
    plumbing only; works with the nccl and gloo backends)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank()
    uid = tp_get_unique_id(transport) if rank == src else b"\0" * 128
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
    dist.broadcast(t, src)
    return bytes(t.cpu().tolist())


def tp_grid_init(mode, world, rank, q=0, d=1, device=0, transport=TP_TRANSPORT_NONE,
                 uid: bytes | None = None):
    m = MODES[mode] if isinstance(mode, str) else int(mode)
    g = C.c_void_p()
    idb = C.create_string_buffer(uid if uid is not None else b"\0" * 128, 128)
    _check(lib.tp_grid_init(C.byref(g), m, world, rank, q, d, device, transport, idb),
           "tp_grid_init")
    return g


def tp_grid_coords(g):
    c = (C.c_int * 3)()
    _check(lib.tp_grid_coords(g, c), "tp_grid_coords")
    return tuple(c)


def tp_grid_dims(g):
    d = (C.c_int * 3)()
    n = C.c_int()
    _check(lib.tp_grid_dims(g, d, C.byref(n)), "tp_grid_dims")
    return tuple(d[: n.value])


def tp_grid_group(g, axis):
    dims = tp_grid_dims(g)
    m = (C.c_int * dims[axis])()
    _check(lib.tp_grid_group(g, axis, m), "tp_grid_group")
    return list(m)


def tp_grid_destroy(g):
    _check(lib.tp_grid_destroy(g), "tp_grid_destroy")


COLLECTIVES = {"bcast": 0, "reduce": 1, "allreduce": 2, "allgather": 3, "reducescatter": 4,
               "shift": 5}


def tp_axis_collective(g, axis, op, send, recv, arg=0, stream=None):
    """One collective over this rank's grid line along `axis` (torch tensors; count = elements
    of send, or of recv for bcast / allgather's per-member slice)."""
    import torch
    o = COLLECTIVES[op] if isinstance(op, str) else int(op)
    dt = DTYPES["bf16"] if recv.dtype == torch.bfloat16 else DTYPES["fp32"]
    src = recv if send is None else send
    count = src.numel() if o != COLLECTIVES["reducescatter"] else recv.numel()
    _check(lib.tp_axis_collective(g, int(axis), o, _ptr(send), _ptr(recv), count, dt, int(arg),
                                  _stream(stream)),
           "tp_axis_collective")


def tp_prof_spans(max_spans=1 << 16):
    """Recorded spans (tp_prof_enable): list of dicts class / rank / start_ms / end_ms / value."""
    buf = (L.tp_span * max_spans)()
    n = C.c_int()
    _check(lib.tp_prof_spans(max_spans, buf, C.byref(n)), "tp_prof_spans")
    return [{"cls": b.kernel_class, "rank": b.rank, "start_ms": b.start_ms, "end_ms": b.end_ms,
             "value": b.value} for b in buf[:min(n.value, max_spans)]]


def tp_peer_staged_bytes(g) -> int:
    """Bytes this rank has pulled from peers by staging copies (TP_FLAG_PEER_STAGED)."""
    v = C.c_uint64()
    _check(lib.tp_peer_staged_bytes(g, C.byref(v)), "tp_peer_staged_bytes")
    return int(v.value)


def tp_knob_set(name, value):
    _check(lib.tp_knob_set(name.encode(), int(value)), "tp_knob_set")


def tp_knob_get(name) -> int:
    v = C.c_int()
    _check(lib.tp_knob_get(name.encode(), C.byref(v)), "tp_knob_get")
    return v.value


def tp_knobs():
    """The library's tuning knobs: list of {name, value, default, source, what}."""
    import json
    need = C.c_size_t()
    _check(lib.tp_knobs(None, 0, C.byref(need)), "tp_knobs")
    buf = C.create_string_buffer(need.value)
    _check(lib.tp_knobs(buf, need.value, C.byref(need)), "tp_knobs")
    return json.loads(buf.value.decode())


def tp_grid_check(g):
    """Raise TPError if a communicator of the grid reports an asynchronous error."""
    _check(lib.tp_grid_check(g), "tp_grid_check")


def tp_grid_abort(g):
    """Abort the grid's communicators (blocked collectives return); destroy-only afterwards."""
    _check(lib.tp_grid_abort(g), "tp_grid_abort")


def tp_grid_set_contract_check(g, enable=True):
    """Debug: verify on every collective call that all ranks passed the same desc (TP_ERR_ARG
    instead of a deadlock on a mismatch)."""
    _check(lib.tp_grid_set_contract_check(g, int(bool(enable))), "tp_grid_set_contract_check")


def tp_shard_extent(g, d: tp_linear_desc, tensor):
    t = TENSORS[tensor] if isinstance(tensor, str) else int(tensor)
    v = [C.c_int64() for _ in range(4)]
    _check(lib.tp_shard_extent(g, C.byref(d), t, *[C.byref(x) for x in v]), "tp_shard_extent")
    return tuple(x.value for x in v)


def tp_workspace_size(g, d: tp_linear_desc):
    ws, sv = C.c_size_t(), C.c_size_t()
    _check(lib.tp_workspace_size(g, C.byref(d), C.byref(ws), C.byref(sv)), "tp_workspace_size")
    return ws.value, sv.value


def _nbytes(t):
    if t is None:
        return 0
    return t.numel() * t.element_size()


def tp_linear_fwd(g, d, x, w, bias, y, saved, ws, stream=None, ws_bytes=None):
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_linear_fwd(g, C.byref(d), _ptr(x), _ptr(w), _ptr(bias), _ptr(y), _ptr(saved),
                             _ptr(ws), wb, _stream(stream)), "tp_linear_fwd")


def tp_linear_bwd(g, d, dy, x, w, saved, dx, dw, dbias, ws, stream=None, ws_bytes=None):
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_linear_bwd(g, C.byref(d), _ptr(dy), _ptr(x), _ptr(w), _ptr(saved), _ptr(dx),
                             _ptr(dw), _ptr(dbias), _ptr(ws), wb, _stream(stream)), "tp_linear_bwd")


def tp_pack(g, d, tensor, global_, shard, stream=None):
    t = TENSORS[tensor] if isinstance(tensor, str) else int(tensor)
    _check(lib.tp_pack(g, C.byref(d), t, _ptr(global_), _ptr(shard), _stream(stream)), "tp_pack")


def tp_unpack(g, d, tensor, shard, global_, stream=None):
    t = TENSORS[tensor] if isinstance(tensor, str) else int(tensor)
    _check(lib.tp_unpack(g, C.byref(d), t, _ptr(shard), _ptr(global_), _stream(stream)),
           "tp_unpack")


def tp_gemm(trans_a, trans_b, M, N, K, in_dtype, A, lda, B, ldb, Cm, ldc, D, ldd, out_dtype,
            alpha=1.0, bias=None, stream=None, ws=None):
    idt = DTYPES[in_dtype] if isinstance(in_dtype, str) else int(in_dtype)
    odt = DTYPES[out_dtype] if isinstance(out_dtype, str) else int(out_dtype)
    _check(lib.tp_gemm(int(trans_a), int(trans_b), M, N, K, idt, _ptr(A), lda, _ptr(B), ldb,
                       _ptr(Cm), ldc, _ptr(D), ldd, odt, float(alpha), _ptr(bias), _ptr(ws),
                       _nbytes(ws), _stream(stream)), "tp_gemm")


def tp_gemm_ws_bytes() -> int:
    return int(lib.tp_gemm_ws_bytes())


def tp_colsum(src, rows, cols, ld, dtype, dst, stream=None):
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    _check(lib.tp_colsum(_ptr(src), rows, cols, ld, dt, _ptr(dst), _stream(stream)), "tp_colsum")


def tp_fill(dst, dtype, rows, cols, ld, seed, tensor_id, kind, scale, g_row0, g_col0, g_cols,
            stream=None):
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    k = {"uniform": 0, "ternary": 1}[kind] if isinstance(kind, str) else int(kind)
    _check(lib.tp_fill(_ptr(dst), dt, rows, cols, ld, seed & 0xFFFFFFFFFFFFFFFF, tensor_id, k,
                       float(scale), g_row0, g_col0, g_cols, _stream(stream)), "tp_fill")


def tp_l2_flush(scratch, stream=None):
    _check(lib.tp_l2_flush(_ptr(scratch), _nbytes(scratch), _stream(stream)), "tp_l2_flush")


def tp_prof_enable(on=True):
    _check(lib.tp_prof_enable(int(bool(on))), "tp_prof_enable")


def tp_prof_reset():
    _check(lib.tp_prof_reset(), "tp_prof_reset")


def tp_prof_read(kernel_class=0):
    ms, fl = C.c_double(), C.c_double()
    n = C.c_int64()
    _check(lib.tp_prof_read(kernel_class, C.byref(ms), C.byref(n), C.byref(fl)), "tp_prof_read")
    return ms.value, n.value, fl.value


def tp_launch_count() -> int:
    return int(lib.tp_launch_count())


def tp_gemm_trace(buf=None):
    _check(lib.tp_gemm_trace(_ptr(buf)), "tp_gemm_trace")


def tp_register_buffer(g, t):
    """Collective: register this rank's copy of a symmetric buffer (torch tensor)."""
    _check(lib.tp_register_buffer(g, _ptr(t), _nbytes(t)), "tp_register_buffer")


def tp_deregister_all(g):
    _check(lib.tp_deregister_all(g), "tp_deregister_all")


def tp_cost_model(mode, world, d_: tp_linear_desc, q=0, depth=1, peak_tflops=0.0, link_gbs=0.0):
    """Analytic per-layer fwd+bwd cost (host only); returns a dict of the tp_cost fields."""
    m = MODES[mode] if isinstance(mode, str) else int(mode)
    c = tp_cost()
    _check(lib.tp_cost_model(m, world, q, depth, C.byref(d_), float(peak_tflops), float(link_gbs),
                             C.byref(c)), "tp_cost_model")
    return {n: getattr(c, n) for n, _ in tp_cost._fields_}


def tp_layernorm_ws_size(g, d, tensor):
    t = TENSORS[tensor] if isinstance(tensor, str) else int(tensor)
    n = C.c_size_t()
    _check(lib.tp_layernorm_ws_size(g, C.byref(d), t, C.byref(n)), "tp_layernorm_ws_size")
    return n.value


def tp_layernorm_fwd(g, d, tensor, eps, x, gamma, beta, y, stats, ws, stream=None, ws_bytes=None):
    t = TENSORS[tensor] if isinstance(tensor, str) else int(tensor)
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_layernorm_fwd(g, C.byref(d), t, float(eps), _ptr(x), _ptr(gamma), _ptr(beta),
                                _ptr(y), _ptr(stats), _ptr(ws), wb, _stream(stream)),
           "tp_layernorm_fwd")


def tp_layernorm_bwd(g, d, tensor, dy, x, gamma, stats, dx, dgamma, dbeta, ws, stream=None,
                     ws_bytes=None):
    t = TENSORS[tensor] if isinstance(tensor, str) else int(tensor)
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_layernorm_bwd(g, C.byref(d), t, _ptr(dy), _ptr(x), _ptr(gamma), _ptr(stats),
                                _ptr(dx), _ptr(dgamma), _ptr(dbeta), _ptr(ws), wb, _stream(stream)),
           "tp_layernorm_bwd")


def rsa_desc(seq, d_k, heads=1, dtype="bf16", scale=0.0) -> tp_rsa_desc:
    dt = DTYPES[dtype] if isinstance(dtype, str) else int(dtype)
    return tp_rsa_desc(int(seq), int(d_k), int(heads), dt, float(scale))


def tp_rsa_ws_size(g, d: tp_rsa_desc) -> int:
    n = C.c_size_t()
    _check(lib.tp_rsa_ws_size(g, C.byref(d), C.byref(n)), "tp_rsa_ws_size")
    return n.value


def tp_rsa_fwd(g, d: tp_rsa_desc, q, k, v, out, ws, stream=None, ws_bytes=None, lse=None):
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_rsa_fwd(g, C.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(ws),
                          wb, _stream(stream)), "tp_rsa_fwd")


def tp_rsa_bwd(g, d: tp_rsa_desc, q, k, v, dout, dq, dk, dv, ws, stream=None, ws_bytes=None,
               out=None, lse=None):
    """out / lse (the forward's, bf16 d_k 64 / 128): the fused ring backward."""
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_rsa_bwd(g, C.byref(d), _ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(dout),
                          _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), wb, _stream(stream)), "tp_rsa_bwd")


def tp_attention_ws_size(g, d, seq, heads) -> int:
    n = C.c_size_t()
    _check(lib.tp_attention_ws_size(g, C.byref(d), int(seq), int(heads), C.byref(n)),
           "tp_attention_ws_size")
    return n.value


def tp_attention_fwd(g, d, seq, heads, qkv, out, ws, scale=0.0, stream=None, ws_bytes=None,
                     lse=None):
    """lse (optional fp32 tensor, heads_local x rows): the forward's row log-sum-exp, which with
    `out` selects the fused backward."""
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_attention_fwd(g, C.byref(d), int(seq), int(heads), float(scale), _ptr(qkv),
                                _ptr(out), _ptr(lse), _ptr(ws), wb, _stream(stream)),
           "tp_attention_fwd")


def tp_attention_bwd(g, d, seq, heads, qkv, dout, dqkv, ws, scale=0.0, stream=None, ws_bytes=None,
                     out=None, lse=None):
    wb = _nbytes(ws) if ws_bytes is None else ws_bytes
    _check(lib.tp_attention_bwd(g, C.byref(d), int(seq), int(heads), float(scale), _ptr(qkv),
                                _ptr(out), _ptr(lse), _ptr(dout), _ptr(dqkv), _ptr(ws), wb,
                                _stream(stream)), "tp_attention_bwd")


def tp_add(a, b, out, dtype=None, stream=None):
    dt = DTYPES[dtype] if isinstance(dtype, str) else (int(dtype) if dtype is not None else
                                                       (TP_BF16 if out.element_size() == 2 else TP_FP32))
    _check(lib.tp_add(_ptr(a), _ptr(b), _ptr(out), out.numel(), dt, _stream(stream)), "tp_add")
