"""ctypes binding of libtp_b200.so (include/tp_b200.h). Argument marshalling only.

The library is built in-tree (python -m paper_2110_14883_b200.build). There is no
fallback: if the .so is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtp_b200.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -m paper_2110_14883_b200.build` "
        "(there is no CPU or PyTorch fallback for the tensor-parallel path)")

lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)

# enums (tp_b200.h)
TP_OK, TP_ERR_CONSTRAINT, TP_ERR_INDIVISIBLE, TP_ERR_SHAPE, TP_ERR_ARG = 0, 1, 2, 3, 4
TP_ERR_CUDA, TP_ERR_NCCL, TP_ERR_WORKSPACE, TP_ERR_UNSUPPORTED = 5, 6, 7, 8
TP_1D, TP_2D, TP_2P5D, TP_3D = 1, 2, 3, 4
TP_BF16, TP_FP32 = 0, 1
TP_TRANSPORT_NCCL, TP_TRANSPORT_LOCAL, TP_TRANSPORT_NONE = 0, 1, 2
TP_TENSOR_X, TP_TENSOR_W, TP_TENSOR_Y, TP_TENSOR_BIAS = 0, 1, 2, 3
TP_FLAG_W25_DEPTH_SHARDED = 0x1
TP_FLAG_SERIAL = 0x2
TP_FLAG_PEER_FUSED = 0x4
TP_FLAG_GELU = 0x8
TP_FLAG_CANNON = 0x10
TP_FLAG_SOLOMONIK = 0x20
TP_FLAG_PEER_STAGED = 0x40

EXPORTED = [
    "tp_status_string", "tp_last_error", "tp_version", "tp_get_unique_id", "tp_grid_init",
    "tp_grid_coords", "tp_grid_dims", "tp_grid_group", "tp_grid_destroy", "tp_shard_extent",
    "tp_knob_set", "tp_knob_get", "tp_knobs", "tp_grid_set_contract_check", "tp_grid_check", "tp_grid_abort", "tp_axis_collective", "tp_peer_staged_bytes", "tp_prof_spans",
    "tp_workspace_size", "tp_linear_fwd", "tp_linear_bwd", "tp_pack", "tp_unpack", "tp_gemm",
    "tp_gemm_ws_bytes",
    "tp_colsum", "tp_fill", "tp_l2_flush", "tp_prof_enable", "tp_prof_reset", "tp_prof_read",
    "tp_launch_count", "tp_gemm_trace", "tp_register_buffer", "tp_deregister_all",
    "tp_cost_model", "tp_layernorm_ws_size", "tp_layernorm_fwd", "tp_layernorm_bwd",
    "tp_rsa_ws_size", "tp_rsa_fwd", "tp_rsa_bwd", "tp_attention_ws_size", "tp_attention_fwd",
    "tp_attention_bwd", "tp_add",
]


class tp_cost(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("paper_elems", "counted_elems", "link_bytes", "flops",
                                          "mem_x", "mem_w", "mem_y", "t_tensor_us", "t_link_us",
                                          "t_roof_us", "t_exposed_us", "fused_direct_bytes",
                                          "fused_staged_bytes")]


class tp_span(C.Structure):
    _fields_ = [("kernel_class", C.c_int), ("rank", C.c_int), ("start_ms", C.c_double),
                ("end_ms", C.c_double), ("value", C.c_double)]


class tp_rsa_desc(C.Structure):
    _fields_ = [("seq", C.c_int64), ("d_k", C.c_int64), ("heads", C.c_int64), ("dtype", C.c_int),
                ("scale", C.c_float)]


class tp_linear_desc(C.Structure):
    _fields_ = [("M", C.c_int64), ("K", C.c_int64), ("N", C.c_int64), ("dtype", C.c_int),
                ("split_1d", C.c_int), ("parity_3d", C.c_int), ("flags", C.c_uint32),
                ("alpha", C.c_float)]


_vp, _i, _i64, _sz, _f = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_float
_P64 = C.POINTER(C.c_int64)

_sigs = {
    "tp_status_string": (C.c_char_p, [_i]),
    "tp_last_error": (C.c_char_p, []),
    "tp_version": (C.c_char_p, []),
    "tp_get_unique_id": (_i, [_i, _vp]),
    "tp_grid_init": (_i, [C.POINTER(_vp), _i, _i, _i, _i, _i, _i, _i, _vp]),
    "tp_grid_coords": (_i, [_vp, C.POINTER(_i)]),
    "tp_grid_dims": (_i, [_vp, C.POINTER(_i), C.POINTER(_i)]),
    "tp_grid_group": (_i, [_vp, _i, C.POINTER(_i)]),
    "tp_grid_destroy": (_i, [_vp]),
    "tp_grid_set_contract_check": (_i, [_vp, _i]),
    "tp_grid_check": (_i, [_vp]),
    "tp_knob_set": (_i, [C.c_char_p, _i]),
    "tp_knob_get": (_i, [C.c_char_p, C.POINTER(_i)]),
    "tp_knobs": (_i, [C.c_char_p, _sz, C.POINTER(_sz)]),
    "tp_grid_abort": (_i, [_vp]),
    "tp_axis_collective": (_i, [_vp, _i, _i, _vp, _vp, _sz, _i, _i, _vp]),
    "tp_peer_staged_bytes": (_i, [_vp, C.POINTER(C.c_uint64)]),
    "tp_prof_spans": (_i, [_i, C.POINTER(tp_span), C.POINTER(_i)]),
    "tp_shard_extent": (_i, [_vp, C.POINTER(tp_linear_desc), _i, _P64, _P64, _P64, _P64]),
    "tp_workspace_size": (_i, [_vp, C.POINTER(tp_linear_desc), C.POINTER(_sz), C.POINTER(_sz)]),
    "tp_linear_fwd": (_i, [_vp, C.POINTER(tp_linear_desc), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "tp_linear_bwd": (_i, [_vp, C.POINTER(tp_linear_desc), _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                           _vp, _sz, _vp]),
    "tp_pack": (_i, [_vp, C.POINTER(tp_linear_desc), _i, _vp, _vp, _vp]),
    "tp_unpack": (_i, [_vp, C.POINTER(tp_linear_desc), _i, _vp, _vp, _vp]),
    "tp_gemm": (_i, [_i, _i, _i64, _i64, _i64, _i, _vp, _i64, _vp, _i64, _vp, _i64, _vp, _i64,
                     _i, _f, _vp, _vp, _sz, _vp]),
    "tp_gemm_ws_bytes": (_sz, []),
    "tp_colsum": (_i, [_vp, _i64, _i64, _i64, _i, _vp, _vp]),
    "tp_fill": (_i, [_vp, _i, _i64, _i64, _i64, C.c_uint64, _i, _i, _f, _i64, _i64, _i64, _vp]),
    "tp_l2_flush": (_i, [_vp, _sz, _vp]),
    "tp_prof_enable": (_i, [_i]),
    "tp_prof_reset": (_i, []),
    "tp_prof_read": (_i, [_i, C.POINTER(C.c_double), _P64, C.POINTER(C.c_double)]),
    "tp_launch_count": (_i64, []),
    "tp_gemm_trace": (_i, [_vp]),
    "tp_register_buffer": (_i, [_vp, _vp, _sz]),
    "tp_deregister_all": (_i, [_vp]),
    "tp_layernorm_ws_size": (_i, [_vp, C.POINTER(tp_linear_desc), _i, C.POINTER(_sz)]),
    "tp_layernorm_fwd": (_i, [_vp, C.POINTER(tp_linear_desc), _i, _f, _vp, _vp, _vp, _vp, _vp, _vp,
                              _sz, _vp]),
    "tp_layernorm_bwd": (_i, [_vp, C.POINTER(tp_linear_desc), _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                              _vp, _sz, _vp]),
    "tp_rsa_ws_size": (_i, [_vp, C.POINTER(tp_rsa_desc), C.POINTER(_sz)]),
    "tp_rsa_fwd": (_i, [_vp, C.POINTER(tp_rsa_desc), _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "tp_rsa_bwd": (_i, [_vp, C.POINTER(tp_rsa_desc), _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                        _vp]),
    "tp_attention_ws_size": (_i, [_vp, C.POINTER(tp_linear_desc), _i64, _i64, C.POINTER(_sz)]),
    "tp_attention_fwd": (_i, [_vp, C.POINTER(tp_linear_desc), _i64, _i64, _f, _vp, _vp, _vp, _vp,
                              _sz, _vp]),
    "tp_attention_bwd": (_i, [_vp, C.POINTER(tp_linear_desc), _i64, _i64, _f, _vp, _vp, _vp, _vp,
                              _vp, _vp, _sz, _vp]),
    "tp_add": (_i, [_vp, _vp, _vp, _sz, _i, _vp]),
    "tp_cost_model": (_i, [_i, _i, _i, _i, C.POINTER(tp_linear_desc), C.c_double, C.c_double,
                           C.POINTER(tp_cost)]),
}

for _name, (_res, _args) in _sigs.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args
