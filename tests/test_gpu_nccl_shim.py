"""Multi-PROCESS worlds on ONE GPU through the library's NCCL transport (TP_TRANSPORT_NCCL), with
tests/ncclshim LD_PRELOADed in place of NCCL (real NCCL rejects two ranks of a communicator on
one device; the test boxes have one GPU).

What runs for real: one process per rank (torch.distributed.run), the id broadcast
(api.share_unique_id over gloo), tp_grid_init's ncclCommInitRank + one ncclCommSplit per grid
line, every grouped collective the 1D / 2D / 2.5D / 3D schedules issue - in the order each rank
issues them (a rank that issued a different sequence would deadlock at the shim's barrier and
fail on its timeout) - and, with TP_FLAG_PEER_FUSED, the CUDA-IPC registration of peer buffers
across processes and the peer-memory panel GEMMs reading another process's shards. Results are
gathered on rank 0 and compared with the dense fp64 oracle (tests/nccl_worker.py).

What the shim replaces: NCCL's data plane (its kernels and NVLink transfers); the shim moves the
bytes through host shared memory (tests/ncclshim/ncclshim.cpp, self-tested on CPU by
tests/test_ncclshim_cpu.py).
"""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))


@pytest.fixture(scope="module")
def shim():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from ncclshim.build import build
    return build()


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_shim_worker(shim, nproc, *args, timeout=600):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "nccl_worker.py"), "--same-gpu", *map(str, args)]
    env = dict(os.environ, LD_PRELOAD=shim, PYTHONPATH=ROOT, TPSHIM_TIMEOUT_S="240",
               TPSHIM_SLOT_MB="256")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-4000:]}"
    return json.loads(lines[-1]), r


GRIDS = [("1d", 2, 1, 0), ("1d", 8, 1, 0), ("2d", 4, 1, 0), ("2d", 9, 1, 0x10), ("2.5d", 8, 2, 0),
         ("2.5d", 8, 2, 0x1), ("2.5d", 8, 2, 0x20), ("3d", 8, 1, 0), ("2d", 4, 1, 0x4),
         ("2.5d", 8, 2, 0x4), ("3d", 8, 1, 0x44)]


@pytest.mark.parametrize("mode,p,d,flags", GRIDS, ids=[f"{m}-p{p}-f{f}" for m, p, _, f in GRIDS])
def test_multiprocess_nccl_transport_one_gpu(shim, mode, p, d, flags):
    """flags: 0x1 depth-sharded 2.5D W, 0x10 Cannon (send/recv shifts), 0x20 Solomonik 2.5D,
    0x4 peer-fused (CUDA IPC), 0x40 with copy-engine staging of the peer panels."""
    M, H = (1024, 512) if flags & 4 else (384, 576)  # 576: divisible by q = 3 and p = 8
    res, r = run_shim_worker(shim, p, "--mode", mode, "--depth", d, "--M", M, "--K", H,
                             "--N", H, "--flags", flags)
    assert res["ok"], (res, r.stderr[-3000:])


def test_multiprocess_contract_check_mismatch_fails_cleanly(shim):
    """Rank 1 passes a different desc with the contract check on: both ranks return TP_ERR_ARG
    (the check's hash all-reduce runs over the NCCL world communicator) instead of hanging."""
    res, r = run_shim_worker(shim, 2, "--mode", "1d", "--M", 256, "--K", 256, "--N", 256,
                             "--contract-check", "--mismatch", timeout=300)
    assert res["statuses"] == ["error", "error"], (res, r.stderr[-3000:])
    assert "contract" in res.get("error", ""), res


def test_multiprocess_contract_check_matching_runs(shim):
    res, r = run_shim_worker(shim, 4, "--mode", "2d", "--M", 256, "--K", 256, "--N", 256,
                             "--contract-check")
    assert res["ok"], (res, r.stderr[-3000:])


BENCH = [(2, "auto", []), (4, "auto", []), (8, "auto", []), (8, "2.5d", []), (4, "auto", ["--fused"])]


@pytest.mark.parametrize("n,mode,extra", BENCH, ids=[f"n{n}-{m}" + "".join(e) for n, m, e in BENCH])
def test_bench_multiprocess_one_gpu(shim, n, mode, extra):
    """bench.py's N > 1 path as the driver launches it (torch.distributed.run, one process per
    rank), all ranks on cuda:0 over the shim: grid init, warm-up, instrumented and timed passes
    (eager launches, the N > 1 default), max over ranks, the e2e arm, the memory and NVLink roof
    fields, one JSON line from rank 0. The timings are meaningless here (host-staged collectives,
    time-sliced GPU); the contract is what is checked."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--steps", "2", "--warmup", "3", "--workload", "c2", "--mode", mode,
           "--no-cpu-baseline", *extra]
    env = dict(os.environ, LD_PRELOAD=shim, PYTHONPATH=ROOT, TPSHIM_TIMEOUT_S="240",
               TPSHIM_SLOT_MB="256", TP_BENCH_DIST_BACKEND="gloo", TP_BENCH_DEVICE="0")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-4000:]}"
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["steps"] == 2 and d["launch"] == "eager"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["grid"] and d["roofline"]["nvlink"]["bytes_per_gpu_per_step"] > 0
    assert d["memory_per_rank"] and d["e2e"]["value"] > 0
    if "--fused" in extra:
        assert d["config"]["parallelism"].endswith("-fused")
