"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic (no matmul, no sharding,
no collective): it only turns (seed, tensor id, element coordinates) into
numbers. Both sides of every parity test draw their inputs from here, or —
on the device — from the CUDA library's own implementation of the SAME
counter-based generator (`tp_fill` in include/tp_b200.h), which is checked
bit-exact against this one.

Generator (SURVEY §8c reading A13; SPEC.md S:L193 names SplitMix64):

  * stream seed   s_t = splitmix64_mix(seed + (tensor_id + 1) * GOLDEN)
  * element (r,c) of a global [rows, cols] tensor uses counter
        i = r * cols + c,   z = splitmix64_mix(s_t + (i + 1) * GOLDEN)
    (this is exactly output i of a SplitMix64 stream seeded with s_t, so
    any element can be drawn independently: shards are generated in place)
  * kind "uniform":  n = z >> 40 (24 bits);  v = f32(n - 2^23) * 2^-23 in [-1, 1)
    exactly, then v = f32(v * f32(scale))  (one IEEE fp32 multiply)
  * kind "ternary":  v = f32((z >> 32) % 3) - 1  in {-1, 0, 1}  (exact-integer pin)
  * the value is then quantised to the storage dtype: bf16 by round-to-nearest-
    even on the fp32 bit pattern, or kept as fp32.

The oracle consumes the QUANTISED values (converted exactly to fp64), so the
only GPU-vs-oracle differences are accumulation order and output rounding.
"""
from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# tensor ids (one independent stream per tensor of a layer)
TID_X, TID_W, TID_DY, TID_BIAS = 0, 1, 2, 3


def layer_tid(layer: int, tid: int) -> int:
    """Stream id of tensor `tid` of layer `layer` (layer 0 = first linear)."""
    return 16 * layer + tid


def _mix(z: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def stream_seed(seed: int, tensor_id: int) -> int:
    with np.errstate(over="ignore"):
        s = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + np.uint64(tensor_id + 1) * GOLDEN
    return int(_mix(np.array([s], dtype=np.uint64))[0])


def raw_u64(seed: int, tensor_id: int, counters: np.ndarray) -> np.ndarray:
    s = np.uint64(stream_seed(seed, tensor_id))
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return _mix(s + (c + np.uint64(1)) * GOLDEN)


def f32_to_bf16_bits(v: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit pattern (uint16). No NaN inputs here."""
    b = np.asarray(v, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = (b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint32) << np.uint32(16)).view(np.float32)


def quantise(v32: np.ndarray, dtype: str) -> np.ndarray:
    """fp32 values -> values exactly representable in `dtype` (returned as fp32)."""
    if dtype == "bf16":
        return bf16_bits_to_f32(f32_to_bf16_bits(v32))
    if dtype == "fp32":
        return np.asarray(v32, dtype=np.float32)
    raise ValueError(dtype)


def values_at(seed: int, tensor_id: int, counters: np.ndarray, kind: str,
              scale: float, dtype: str) -> np.ndarray:
    """Generator output at the given flat counters, quantised, as fp32."""
    z = raw_u64(seed, tensor_id, counters)
    if kind == "uniform":
        n = (z >> np.uint64(40)).astype(np.int64) - (1 << 23)
        v = n.astype(np.float32) * np.float32(2.0 ** -23)
        v = (v * np.float32(scale)).astype(np.float32)
    elif kind == "ternary":
        v = ((z >> np.uint64(32)) % np.uint64(3)).astype(np.float32) - np.float32(1.0)
    else:
        raise ValueError(kind)
    return quantise(v, dtype)


_PAR_MIN = 1 << 22      # elements above which tensor() splits its rows over threads


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


def tensor(seed: int, tensor_id: int, rows: int, cols: int, kind: str = "uniform",
           scale: float = 1.0, dtype: str = "bf16", row0: int = 0, nrows: int | None = None,
           col0: int = 0, ncols: int | None = None) -> np.ndarray:
    """Block [row0:row0+nrows, col0:col0+ncols] of the global [rows, cols] tensor, fp32.

    Large blocks are generated as row chunks on a thread pool (numpy releases the GIL in its
    ufuncs); every element depends only on its own counter, so the values are identical."""
    nrows = rows - row0 if nrows is None else nrows
    ncols = cols - col0 if ncols is None else ncols
    c = np.arange(col0, col0 + ncols, dtype=np.uint64)[None, :]

    def block(r_lo, r_hi):
        r = np.arange(r_lo, r_hi, dtype=np.uint64)[:, None]
        return values_at(seed, tensor_id, r * np.uint64(cols) + c, kind, scale, dtype)

    nt = _threads()
    if nrows * ncols < _PAR_MIN or nt == 1 or nrows < 2:
        return block(row0, row0 + nrows).reshape(nrows, ncols)
    out = np.empty((nrows, ncols), dtype=np.float32)
    step = max(1, min(nrows, (1 << 20) // max(ncols, 1)))

    def fill(lo):
        hi = min(nrows, lo + step)
        out[lo:hi] = block(row0 + lo, row0 + hi)

    with ThreadPoolExecutor(nt) as ex:
        list(ex.map(fill, range(0, nrows, step)))
    return out


def rows_of(seed, tensor_id, rows, cols, row_idx, kind="uniform", scale=1.0, dtype="bf16"):
    """Selected full rows of the global tensor (sampled oracle)."""
    r = np.asarray(row_idx, dtype=np.uint64)[:, None]
    c = np.arange(cols, dtype=np.uint64)[None, :]
    return values_at(seed, tensor_id, r * np.uint64(cols) + c, kind, scale, dtype)


def cols_of(seed, tensor_id, rows, cols, col_idx, kind="uniform", scale=1.0, dtype="bf16"):
    """Selected full columns of the global tensor, shape [rows, len(col_idx)]."""
    r = np.arange(rows, dtype=np.uint64)[:, None]
    c = np.asarray(col_idx, dtype=np.uint64)[None, :]
    return values_at(seed, tensor_id, r * np.uint64(cols) + c, kind, scale, dtype)


def xavier_scale(fan_in: int, fan_out: int) -> float:
    """Xavier-uniform bound sqrt(6/(fan_in+fan_out)) ("Jax initialization")."""
    return math.sqrt(6.0 / (fan_in + fan_out))


# --- workload recipes ---------------------------------------

def layer_inputs(seed: int, M: int, K: int, N: int, layer: int = 0, kind: str = "uniform",
                 dtype: str = "bf16", with_bias: bool = False):
    """Global X [M,K], W [K,N], dY [M,N] (and bias [N]) of one linear layer, fp32 arrays."""
    ws = xavier_scale(K, N) if kind == "uniform" else 1.0
    X = tensor(seed, layer_tid(layer, TID_X), M, K, kind, 1.0, dtype)
    W = tensor(seed, layer_tid(layer, TID_W), K, N, kind, ws, dtype)
    dY = tensor(seed, layer_tid(layer, TID_DY), M, N, kind, 1.0, dtype)
    b = tensor(seed, layer_tid(layer, TID_BIAS), 1, N, kind, 1.0, dtype)[0] if with_bias else None
    return X, W, dY, b
