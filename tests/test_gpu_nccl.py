"""The NCCL transport (TP_TRANSPORT_NCCL) and the collective-contract check, on one B200.

* Every mode's 1-rank grid through TP_TRANSPORT_NCCL in this process (ncclGetUniqueId,
  ncclCommInitRank, the schedules' p = 1 paths) against the dense oracle.
* Every collective of the NCCL wrappers (tp_axis_collective on 1-rank NCCL lines: the ncclBroadcast
  / Reduce / AllReduce / AllGather / ReduceScatter / Send+Recv calls, their counts, dtypes and
  in-place conventions) and of the LOCAL transport on 2-, 4- and 8-rank lines, against the
  oracle's simulated collectives (oracle/fabric.py).
* Multi-process NCCL worlds, one rank per GPU (tests/nccl_worker.py under
  torch.distributed.run): ncclCommInitRank + ncclCommSplit per grid line, the grouped
  collectives of the 1D / 2D / 2.5D / 3D schedules, and with TP_FLAG_PEER_FUSED the CUDA-IPC
  buffer registration and peer-memory panel GEMMs - compared with the dense fp64 oracle on
  rank 0. NCCL rejects two ranks on one GPU, so these skip on boxes with fewer GPUs than ranks.
* The collective-contract check (tp_grid_set_contract_check): mismatched descs
  return TP_ERR_ARG on every rank instead of deadlocking (LOCAL and NCCL transports).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth
from tp_harness import (chain_reference, gather, oracle_layer, rel_fro, run_ranks, spec_of,
                        tp_layer)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def api():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2110_14883_b200 import api
    return api


@pytest.mark.parametrize("mode", ["1d", "2d", "2.5d", "3d"])
def test_nccl_transport_one_rank_every_mode(api, mode):
    from paper_2110_14883_b200.mlp import TPMLP
    M, layers = 256, [(384, 256), (256, 128)]
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_NCCL)
    g = api.tp_grid_init(mode, 1, 0, 0, 1, 0, api.TP_TRANSPORT_NCCL, uid)
    try:
        m = TPMLP(g, M, layers, seed=5)
        m.step()
        torch.cuda.synchronize()
        got = (m.Y[-1], m.dX[0], m.dW[0], m.dW[1])
        got = [t.float().cpu().numpy() for t in got]
    finally:
        api.tp_grid_destroy(g)
    for a, b in zip(got, chain_reference(5, M, layers)):
        assert rel_fro(a, b) <= 1e-2


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_worker(nproc, *args, timeout=300):
    """NCCL refuses two ranks of one communicator on the same GPU ("Duplicate GPU detected",
    ncclInvalidUsage - measured on the B200 boxes), so a p-rank NCCL world needs p GPUs."""
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"{nproc}-rank NCCL world needs {nproc} GPUs (NCCL rejects duplicate GPUs); "
                    f"this box has {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "nccl_worker.py"), *map(str, args)]
    env = dict(os.environ, NCCL_DEBUG="WARN", PYTHONPATH=ROOT)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, f"rc={r.returncode}\n{r.stdout[-3000:]}\n{r.stderr[-3000:]}"
    return json.loads(lines[-1]), r


NCCL_GRIDS = [("1d", 2, 1, 0), ("1d", 4, 1, 0), ("2d", 4, 1, 0), ("2.5d", 8, 2, 0),
              ("2.5d", 8, 2, 1), ("3d", 8, 1, 0), ("2d", 4, 1, 4), ("3d", 8, 1, 4)]


@pytest.mark.parametrize("mode,p,d,flags", NCCL_GRIDS,
                         ids=[f"{m}-p{p}-f{f}" for m, p, _, f in NCCL_GRIDS])
def test_nccl_multiprocess(api, mode, p, d, flags):
    M = 1024 if flags & 4 else 256  # the fused panel GEMMs need blocks > 128 rows
    res, r = run_worker(p, "--mode", mode, "--depth", d, "--M", M, "--K", 512, "--N", 512,
                        "--flags", flags)
    assert res["ok"], (res, r.stderr[-3000:])


def test_nccl_contract_check_mismatch_fails_cleanly(api):
    res, r = run_worker(2, "--mode", "1d", "--M", 256, "--K", 256, "--N", 256, "--contract-check",
                        "--mismatch", timeout=180)
    assert res["statuses"] == ["error", "error"], res
    assert "contract" in res.get("error", ""), res


def test_nccl_contract_check_matching_runs(api):
    res, r = run_worker(4, "--mode", "2d", "--M", 256, "--K", 256, "--N", 256, "--contract-check")
    assert res["ok"], (res, r.stderr[-3000:])


def test_local_contract_check_mismatch_fails_cleanly(api):
    """LOCAL transport, 1D p=2: rank 1 passes a different M; both ranks get TP_ERR_ARG, nothing
    is enqueued, no rank hangs (run_ranks times out otherwise)."""
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)

    def rank_fn(r):
        g = api.tp_grid_init("1d", 2, r, 0, 1, 0, api.TP_TRANSPORT_LOCAL, uid)
        try:
            api.tp_grid_set_contract_check(g, True)
            M = 128 if r == 0 else 256
            ds = api.desc(M, 128, 128)
            wsb, _ = api.tp_workspace_size(g, ds)
            ext = {t: api.tp_shard_extent(g, ds, t) for t in ("X", "W", "Y")}
            mk = lambda t: torch.zeros(ext[t][1], ext[t][3], device="cuda", dtype=torch.bfloat16)
            ws = torch.empty(max(wsb, 1), device="cuda", dtype=torch.uint8)
            n0 = api.tp_launch_count()
            try:
                api.tp_linear_fwd(g, ds, mk("X"), mk("W"), None, mk("Y"), None, ws)
            except api.TPError as e:
                return str(e), api.tp_launch_count() - n0
            return "ran", 0
        finally:
            api.tp_grid_destroy(g)

    res = run_ranks(2, rank_fn, timeout=60)
    for msg, _ in res:
        assert "contract" in msg, res


def test_local_contract_check_kind_mismatch(api):
    """Rank 0 calls fwd, rank 1 calls bwd with the same desc: TP_ERR_ARG on both."""
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)

    def rank_fn(r):
        g = api.tp_grid_init("1d", 2, r, 0, 1, 0, api.TP_TRANSPORT_LOCAL, uid)
        try:
            api.tp_grid_set_contract_check(g, True)
            ds = api.desc(128, 128, 128)
            wsb, _ = api.tp_workspace_size(g, ds)
            ext = {t: api.tp_shard_extent(g, ds, t) for t in ("X", "W", "Y")}
            mk = lambda t: torch.zeros(ext[t][1], ext[t][3], device="cuda", dtype=torch.bfloat16)
            ws = torch.empty(max(wsb, 1), device="cuda", dtype=torch.uint8)
            try:
                if r == 0:
                    api.tp_linear_fwd(g, ds, mk("X"), mk("W"), None, mk("Y"), None, ws)
                else:
                    api.tp_linear_bwd(g, ds, mk("Y"), mk("X"), mk("W"), None, mk("X"), mk("W"),
                                      None, ws)
            except api.TPError as e:
                return str(e)
            return "ran"
        finally:
            api.tp_grid_destroy(g)

    res = run_ranks(2, rank_fn, timeout=60)
    assert all("contract" in m for m in res), res


@pytest.mark.parametrize("mode,p,d", [("1d", 2, 1), ("2d", 4, 1), ("3d", 8, 1)])
def test_local_contract_check_matching_descs_unchanged(api, mode, p, d):
    """With the check on and identical descs, the results equal the oracle as without it."""
    M, K, N = 64, 128, 64
    X, W, dY, _ = synth.layer_inputs(9, M, K, N)
    per = tp_layer_checked(api, mode, p, d, M, K, N, X, W, dY)
    spec = spec_of(M, K, N)
    ref = oracle_layer(mode, p, d, spec, X, W, dY)
    for (key, t), r in zip((("Y", "Y"), ("dX", "X"), ("dW", "W")), ref):
        assert rel_fro(gather(mode, p, d, spec, per, key, t), r) <= 1e-2


def tp_layer_checked(api, mode, p, d, M, K, N, X, W, dY):
    orig = api.tp_grid_init

    def init_checked(*a, **k):
        g = orig(*a, **k)
        api.tp_grid_set_contract_check(g, True)
        return g

    api.tp_grid_init = init_checked
    try:
        return tp_layer(api, mode, p, d, M, K, N, X, W, dY)
    finally:
        api.tp_grid_init = orig


# ------------------------------------------------------------------ line collectives vs fabric

def _expected_collective(op, parts, arg, pos):
    """oracle/fabric.py's simulated collective for a line whose members (positions 0..n-1) hold
    `parts`; returns what member `pos` receives."""
    from oracle.fabric import Fabric
    fab = Fabric()
    n = len(parts)
    group = list(range(n))
    P = {r: parts[r] for r in group}
    if op == "bcast":
        return fab.broadcast(group, arg, P[arg])[pos]
    if op == "reduce":
        return fab.reduce(group, arg, P) if pos == arg else None
    if op == "allreduce":
        return fab.all_reduce(group, P)[pos]
    if op == "allgather":
        return fab.all_gather(group, P)[pos]
    if op == "reducescatter":
        return fab.reduce_scatter(group, P)[pos]
    if op == "shift":
        return parts[(pos + arg) % n]
    raise ValueError(op)


OPS = [("bcast", 1), ("reduce", 0), ("allreduce", 0), ("allgather", 0), ("reducescatter", 0),
       ("shift", -1), ("shift", 1)]


def _line_values(rank, count, op):
    n_in = count * 8 if op == "reducescatter" else count
    return synth.tensor(3, 100 + rank, 1, n_in, kind="ternary", dtype="fp32")[0]


@pytest.mark.parametrize("mode,p,d", [("1d", 2, 1), ("2d", 4, 1), ("3d", 8, 1)])
def test_local_axis_collectives_match_fabric(api, mode, p, d):
    """Every op on every axis of a LOCAL in-process grid (exact integer data, fp32)."""
    from oracle.grid import build_grid
    og = build_grid(mode, p, d)
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)
    count = 96

    def rank_fn(r):
        g = api.tp_grid_init(mode, p, r, 0, d, 0, api.TP_TRANSPORT_LOCAL, uid)
        s = torch.cuda.Stream()
        out = {}
        try:
            with torch.cuda.stream(s):
                for ax in range(len(og.dims)):
                    members = og.group(r, ax)
                    n = len(members)
                    for op, arg in OPS:
                        if op == "bcast" or op == "reduce":
                            arg = min(arg, n - 1)
                        v = _line_values(r, count, op)
                        send = torch.from_numpy(v).cuda()
                        if op == "bcast":
                            recv = send.clone()
                            api.tp_axis_collective(g, ax, op, None, recv, arg)
                        else:
                            m = {"allgather": count * n, "reducescatter": count * 8 // n}.get(op, count)
                            recv = torch.full((m,), float("nan"), device="cuda")
                            if op == "reducescatter":
                                send = send[: count * 8 // n * n].contiguous()
                            api.tp_axis_collective(g, ax, op, send, recv, arg)
                        out[(ax, op, arg)] = recv.cpu().numpy()
            s.synchronize()
            return out
        finally:
            s.synchronize()
            api.tp_grid_destroy(g)

    res = run_ranks(p, rank_fn, timeout=120)
    for r in range(p):
        for ax in range(len(og.dims)):
            members = og.group(r, ax)
            n, pos = len(members), og.group(r, ax).index(r)
            for op, arg in OPS:
                if op in ("bcast", "reduce"):
                    arg = min(arg, n - 1)
                parts = [_line_values(m, count, op) for m in members]
                if op == "reducescatter":
                    parts = [x[: count * 8 // n * n] for x in parts]
                exp = _expected_collective(op, [x.astype(np.float64) for x in parts], arg, pos)
                if exp is None:
                    continue
                got = res[r][(ax, op, arg)]
                assert np.array_equal(got, np.asarray(exp, np.float64).ravel()), (r, ax, op, arg)


@pytest.mark.parametrize("dt", ["fp32", "bf16"])
def test_nccl_axis_collectives_one_rank_lines(api, dt):
    """World 1 over NCCL: every op on a 1-rank NCCL communicator per axis of a 3D l=1 grid -
    the wrappers' NCCL calls run (identity semantics)."""
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_NCCL)
    g = api.tp_grid_init("3d", 1, 0, 0, 1, 0, api.TP_TRANSPORT_NCCL, uid)
    tdt = torch.float32 if dt == "fp32" else torch.bfloat16
    try:
        for ax in range(3):
            for op, arg in OPS:
                v = torch.from_numpy(_line_values(ax, 4096, "x")).cuda().to(tdt)
                if op == "bcast":
                    recv = v.clone()
                    api.tp_axis_collective(g, ax, op, None, recv, 0)
                else:
                    recv = torch.full_like(v, float("nan"))
                    api.tp_axis_collective(g, ax, op, v, recv, 0 if op == "reduce" else arg)
                torch.cuda.synchronize()
                assert torch.equal(recv, v), (ax, op)
    finally:
        api.tp_grid_destroy(g)


def test_grid_check_and_abort(api):
    """Failure detection: tp_grid_check is TP_OK on healthy grids (NCCL and LOCAL); after
    tp_grid_abort the NCCL grid can still be destroyed."""
    uid = api.tp_get_unique_id(api.TP_TRANSPORT_NCCL)
    g = api.tp_grid_init("3d", 1, 0, 0, 1, 0, api.TP_TRANSPORT_NCCL, uid)
    try:
        api.tp_grid_check(g)
        x = torch.ones(256, device="cuda")
        y = torch.empty_like(x)
        api.tp_axis_collective(g, 0, "allreduce", x, y)  # a 1-rank NCCL line communicator
        torch.cuda.synchronize()
        api.tp_grid_check(g)
        api.tp_grid_abort(g)
    finally:
        api.tp_grid_destroy(g)
    uidl = api.tp_get_unique_id(api.TP_TRANSPORT_LOCAL)

    def rank_fn(r):
        gl = api.tp_grid_init("2d", 4, r, 0, 1, 0, api.TP_TRANSPORT_LOCAL, uidl)
        try:
            api.tp_grid_check(gl)
            return True
        finally:
            api.tp_grid_destroy(gl)

    assert all(run_ranks(4, rank_fn, timeout=60))
