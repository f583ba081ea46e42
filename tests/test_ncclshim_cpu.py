"""CPU self-test of tests/ncclshim (the one-GPU multi-process NCCL stand-in used by
test_gpu_nccl_shim.py): with TPSHIM_HOST_BUFFERS=1 the shim works on host buffers, so p plain
processes can check its rendezvous (ncclCommInitRank on a shared id, ncclCommSplit with colors,
keys and NCCL_SPLIT_NOCOLOR), every collective (fp32 / bf16 / int32, in place and not), grouped
send/recv shifts and group deferral against values computed here from the inputs.
"""
import ctypes as C
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

INT32, F32, BF16 = 2, 7, 9


class UID(C.Structure):
    _fields_ = [("internal", C.c_char * 128)]


def _lib(path):
    lib = C.CDLL(path)
    for f in ("ncclBroadcast", "ncclReduce", "ncclAllReduce", "ncclReduceScatter", "ncclAllGather",
              "ncclSend", "ncclRecv", "ncclCommSplit", "ncclCommInitRank", "ncclGroupStart",
              "ncclGroupEnd", "ncclCommDestroy", "ncclGetUniqueId"):
        getattr(lib, f).restype = C.c_int
    lib.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, UID, C.c_int]
    return lib


def _bf16(x):
    """float32 -> bf16 bits (round to nearest even) and back, numpy."""
    u = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _f(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32)


def _values(rank, n, dt):
    rng = np.random.default_rng(100 + rank)
    if dt == INT32:
        return rng.integers(-50, 50, n).astype(np.int32)
    v = rng.uniform(-1, 1, n).astype(np.float32)
    return _bf16(v) if dt == BF16 else v


def _sum(parts, dt):
    if dt == INT32:
        return np.sum(parts, axis=0).astype(np.int32)
    acc = np.zeros(parts[0].shape, np.float32)
    for x in parts:
        acc += _f(x) if dt == BF16 else x
    return _bf16(acc) if dt == BF16 else acc


def _ptr(a):
    return C.c_void_p(a.ctypes.data)


def _rank_main(path, world, rank, uid, q):
    os.environ["TPSHIM_HOST_BUFFERS"] = "1"
    os.environ["TPSHIM_SLOT_MB"] = "4"
    os.environ["TPSHIM_TIMEOUT_S"] = "60"
    lib = _lib(path)
    try:
        comm = C.c_void_p()
        u = UID()
        u.internal = uid
        assert lib.ncclCommInitRank(C.byref(comm), world, u, rank) == 0
        # split: color = rank % 2, key = -rank (reverses the order), rank 3 opts out
        color = -1 if rank == 3 else rank % 2
        sub = C.c_void_p()
        assert lib.ncclCommSplit(comm, color, -rank, C.byref(sub), None) == 0
        members = [r for r in range(world) if r != 3 and r % 2 == rank % 2]
        members.sort(key=lambda r: -r)
        res = {}
        lines = [("world", comm, list(range(world)))]
        if color >= 0:
            lines.append(("split", sub, members))
        else:
            res["nocolor_null"] = sub.value is None
        n = 48
        for name, c, mem in lines:
            p, pos = len(mem), mem.index(rank)
            for dt in (F32, BF16, INT32):
                mine = _values(rank, n * p, dt)
                parts = [_values(r, n * p, dt) for r in mem]
                # all-reduce (out of place) and in place
                out = np.zeros_like(mine)
                assert lib.ncclAllReduce(_ptr(mine), _ptr(out), C.c_size_t(n * p), dt, 0, c, None) == 0
                res[(name, dt, "allreduce")] = np.array_equal(out, _sum(parts, dt))
                buf = mine.copy()
                assert lib.ncclAllReduce(_ptr(buf), _ptr(buf), C.c_size_t(n * p), dt, 0, c, None) == 0
                res[(name, dt, "allreduce_inplace")] = np.array_equal(buf, _sum(parts, dt))
                # broadcast from the last position, in place
                buf = mine.copy()
                assert lib.ncclBroadcast(_ptr(buf), _ptr(buf), C.c_size_t(n * p), dt, p - 1, c, None) == 0
                res[(name, dt, "bcast")] = np.array_equal(buf, parts[p - 1])
                # reduce to position 0
                out = np.zeros_like(mine)
                assert lib.ncclReduce(_ptr(mine), _ptr(out), C.c_size_t(n * p), dt, 0, 0, c, None) == 0
                if pos == 0:
                    res[(name, dt, "reduce")] = np.array_equal(out, _sum(parts, dt))
                # all-gather (in place: send = own block of recv)
                out = np.zeros(n * p, mine.dtype)
                out[pos * n:(pos + 1) * n] = mine[:n]
                snd = out[pos * n:(pos + 1) * n]
                assert lib.ncclAllGather(_ptr(snd), _ptr(out), C.c_size_t(n), dt, c, None) == 0
                res[(name, dt, "allgather")] = np.array_equal(out, np.concatenate([x[:n] for x in parts]))
                # reduce-scatter
                out = np.zeros(n, mine.dtype)
                assert lib.ncclReduceScatter(_ptr(mine), _ptr(out), C.c_size_t(n), dt, 0, c, None) == 0
                res[(name, dt, "reducescatter")] = np.array_equal(out, _sum(parts, dt)[pos * n:(pos + 1) * n])
            # grouped shift by +1 (send to pos-1, receive from pos+1) and two grouped collectives
            mine = _values(rank, n, F32)
            out = np.zeros_like(mine)
            assert lib.ncclGroupStart() == 0
            assert lib.ncclSend(_ptr(mine), C.c_size_t(n), F32, (pos - 1) % p, c, None) == 0
            assert lib.ncclRecv(_ptr(out), C.c_size_t(n), F32, (pos + 1) % p, c, None) == 0
            assert lib.ncclGroupEnd() == 0
            res[(name, "shift")] = np.array_equal(out, _values(mem[(pos + 1) % p], n, F32))
            a, b = mine.copy(), mine.copy()
            assert lib.ncclGroupStart() == 0
            assert lib.ncclAllReduce(_ptr(a), _ptr(a), C.c_size_t(n), F32, 0, c, None) == 0
            assert lib.ncclBroadcast(_ptr(b), _ptr(b), C.c_size_t(n), F32, 0, c, None) == 0
            res[(name, "deferred")] = np.array_equal(a, mine)  # nothing ran inside the group
            assert lib.ncclGroupEnd() == 0
            res[(name, "group")] = (np.array_equal(a, _sum([_values(r, n, F32) for r in mem], F32))
                                    and np.array_equal(b, _values(mem[0], n, F32)))
        if color >= 0:
            lib.ncclCommDestroy(sub)
        lib.ncclCommDestroy(comm)
        q.put((rank, {str(k): bool(v) for k, v in res.items()}))
    except BaseException as e:  # noqa: BLE001
        q.put((rank, {"error": repr(e)}))


@pytest.fixture(scope="module")
def shim():
    from ncclshim.build import build
    return build()


@pytest.mark.parametrize("world", [4, 6])
def test_shim_collectives_and_split(shim, world):
    lib = _lib(shim)
    u = UID()
    assert lib.ncclGetUniqueId(C.byref(u)) == 0
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_rank_main, args=(shim, world, r, u.internal, q)) for r in range(world)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(30)
    for r in range(world):
        assert "error" not in got[r], got[r]
        bad = [k for k, v in got[r].items() if not v]
        assert not bad, (r, bad)
        assert len(got[r]) >= (19 if r == 3 else 36), len(got[r])
