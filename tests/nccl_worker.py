"""One rank of a multi-process TP_TRANSPORT_NCCL run (test helper, launched by
tests/test_gpu_nccl.py through torch.distributed.run; not collected by pytest).

Every rank: gloo process group for the rendezvous only, the 128-byte NCCL id broadcast
(api.share_unique_id), tp_grid_init over NCCL (ncclCommInitRank + ncclCommSplit per grid line),
optional collective-contract check, the two-layer step through TPMLP (the schedules' grouped
NCCL broadcasts / reduces / all-gathers / reduce-scatters / all-reduces, or with --fused the
CUDA-IPC registration and peer-memory panel GEMMs), then the shards are gathered on rank 0 and
compared with the dense fp64 oracle (test infrastructure). Rank 0 prints one JSON line.

    python -m torch.distributed.run --nproc-per-node P --master-addr 127.0.0.1 \
        --master-port PORT tests/nccl_worker.py --mode 2d --M 256 --K 256 --N 256 [--same-gpu]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="1d")
    ap.add_argument("--depth", type=int, default=1)
    ap.add_argument("--M", type=int, default=256)
    ap.add_argument("--K", type=int, default=256)
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--same-gpu", action="store_true", help="every rank on cuda:0")
    ap.add_argument("--contract-check", action="store_true")
    ap.add_argument("--mismatch", action="store_true",
                    help="rank 1 passes a different M (with --contract-check: must fail cleanly)")
    a = ap.parse_args()

    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2110_14883_b200 import api
    from paper_2110_14883_b200.mlp import TPMLP

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = 0 if a.same_gpu else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    out = {"rank": rank, "world": world, "ok": False}
    try:
        uid = api.share_unique_id(api.TP_TRANSPORT_NCCL)
        g = api.tp_grid_init(a.mode, world, rank, 0, a.depth, dev, api.TP_TRANSPORT_NCCL, uid)
        if a.contract_check:
            api.tp_grid_set_contract_check(g, True)
        layers = [(a.K, a.N)] + [(a.N, a.N)] * (a.layers - 1)
        M = a.M * (2 if (a.mismatch and rank == 1) else 1)
        m = TPMLP(g, M, layers, seed=5, flags=a.flags)
        try:
            m.step()
            torch.cuda.synchronize()
            out["status"] = "ran"
        except api.TPError as e:
            out["status"] = "error"
            out["error"] = str(e)
        shards = None
        if out["status"] == "ran":
            shards = {"Y": m.Y[-1].float().cpu().numpy(), "dX": m.dX[0].float().cpu().numpy(),
                      "dW": [w.float().cpu().numpy() for w in m.dW]}
        allsh = [None] * world
        dist.all_gather_object(allsh, shards)
        statuses = [None] * world
        dist.all_gather_object(statuses, out.get("status"))
        out["statuses"] = statuses
        api.tp_grid_destroy(g)
        if rank == 0 and all(s is not None for s in allsh):
            import synth
            from oracle import dense
            from oracle.grid import build_grid
            from oracle.shards import LayerSpec, gather_full
            from tp_harness import rel_fro
            X = synth.tensor(5, synth.layer_tid(0, 0), a.M, layers[0][0]).astype(np.float64)
            Ws = [synth.tensor(5, synth.layer_tid(i, 1), K, N, scale=synth.xavier_scale(K, N))
                  .astype(np.float64) for i, (K, N) in enumerate(layers)]
            dY = synth.tensor(5, synth.layer_tid(len(layers) - 1, 2), a.M, layers[-1][1]
                              ).astype(np.float64)
            acts = [X]
            for W in Ws:
                acts.append(dense.linear_fwd(acts[-1], W))
            d, dWs = dY, [None] * len(Ws)
            for i in reversed(range(len(Ws))):
                d, dWs[i], _ = dense.linear_bwd(d, acts[i], Ws[i])
            og = build_grid(a.mode, world, a.depth)
            if a.flags & api.TP_FLAG_SOLOMONIK:  # Solomonik 2.5D keeps its own shard layout
                from oracle import solomonik as so
                gather_full = lambda g_, sp, sh, t: so.gather_full(g_, sp, sh, t)  # noqa: E731
            sharded = bool(a.flags & api.TP_FLAG_W25_DEPTH_SHARDED)
            specs = [LayerSpec(a.M, K, N, split_1d="row" if i % 2 else "col", parity=i % 2,
                               w_depth_sharded=sharded) for i, (K, N) in enumerate(layers)]
            errs = {"Y": rel_fro(gather_full(og, specs[-1], {r: allsh[r]["Y"] for r in range(world)},
                                             "Y"), acts[-1]),
                    "dX": rel_fro(gather_full(og, specs[0], {r: allsh[r]["dX"] for r in range(world)},
                                              "X"), d)}
            for i in range(len(layers)):
                errs[f"dW{i}"] = rel_fro(gather_full(og, specs[i],
                                                     {r: allsh[r]["dW"][i] for r in range(world)},
                                                     "W"), dWs[i])
            out["errs"] = errs
            out["ok"] = all(v <= 1e-2 for v in errs.values())
        elif rank == 0:
            out["ok"] = False
    finally:
        if rank == 0:
            print(json.dumps(out), flush=True)
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
