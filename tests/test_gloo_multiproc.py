"""Multi-process host logic of the N > 1 path on CPU (gloo, world_size 2 and 4): the 128-byte
rendezvous id broadcast, every rank's grid view (coords, groups) and shard extents agree with
each other and with the oracle, and the max-over-ranks timing reduction (bench contract)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, depth, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2110_14883_b200 import api
    from oracle.grid import build_grid
    from oracle.shards import LayerSpec, extent

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        uid = api.share_unique_id(api.TP_TRANSPORT_LOCAL)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert all(i == ids[0] for i in ids) and uid[:8] != b"\0" * 8
        g = api.tp_grid_init(mode, world, rank, 0, depth)
        og = build_grid(mode, world, depth)
        M, K, N = 8 * world, 16 * world, 8 * world
        ds = api.desc(M, K, N)
        view = {"coords": api.tp_grid_coords(g)[: len(og.dims)],
                "groups": [api.tp_grid_group(g, a) for a in range(len(og.dims))],
                "ext": {t: api.tp_shard_extent(g, ds, t) for t in ("X", "W", "Y", "B")}}
        api.tp_grid_destroy(g)
        views = [None] * world
        dist.all_gather_object(views, view)
        coords = [tuple(v["coords"]) for v in views]
        assert len(set(coords)) == world                       # bijection rank <-> coords
        spec = LayerSpec(M, K, N)
        for r, v in enumerate(views):
            assert tuple(v["coords"]) == og.coords(r)
            for a, grp in enumerate(v["groups"]):
                assert grp == og.group(r, a)
                for m in grp:                                   # members see the same group
                    assert views[m]["groups"][a] == grp
            for t, e in v["ext"].items():
                oe = extent(og, spec, r, t)
                assert tuple(e) == (oe.row0, oe.rows, oe.col0, oe.cols)
        # bench timing contract: max over ranks
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.item() == world
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,depth", [(2, "1d", 1), (4, "2d", 1), (4, "2.5d", 1),
                                              (8, "3d", 1), (8, "2.5d", 2)])
def test_multiprocess_grid_agreement(world, mode, depth):
    from paper_2110_14883_b200 import build
    build.build()
    mp.start_processes(_worker, args=(world, _free_port(), mode, depth, 0), nprocs=world,
                       join=True, start_method="spawn")
