"""Multi-process (world_size 2, gloo, CPU) checks of the multi-GPU host logic: NCCL-id bootstrap
over torch.distributed and the slab partition every rank derives independently."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_15249_b200 import KFBI, broadcast_unique_id
        nid = broadcast_unique_id()
        k = KFBI(W.C3(2048), workspace=False, world=world, rank=rank, nccl_id=nid)
        sl = k.slab()
        stencil = k.setup_dump(2).reshape(-1, 2)[:, 0]           # columns of all stencil nodes
        owned = int(((stencil >= sl["col_lo"]) & (stencil <= sl["col_hi"])).sum())
        out = [None] * world
        k1 = KFBI(W.C3(2048), workspace=False)
        dist.all_gather_object(out, (nid, sl, owned, int(stencil.size), k.local_offset, k.local_shape,
                                     k.workspace_bytes, k1.workspace_bytes))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_partition_and_id_bootstrap(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ids = {r[0] for r in res}
    assert len(ids) == 1 and len(next(iter(ids))) == 128           # one NCCL id, seen by every rank
    slabs = [r[1] for r in res]
    n = 2048
    # blocks, columns and stencil columns tile their ranges disjointly and completely, in rank order
    assert slabs[0]["g_lo"] == 0 and slabs[-1]["g_hi"] == n // 16
    assert slabs[0]["col_lo"] == 1 and slabs[-1]["col_hi"] == n - 1
    assert slabs[0]["o_lo"] == 0
    for a, b in zip(slabs[:-1], slabs[1:]):
        assert a["g_hi"] == b["g_lo"] and a["col_hi"] + 1 == b["col_lo"] and a["o_hi"] == b["o_lo"]
        assert (a["g_hi"] * 16) == a["col_hi"]                       # slab ends on a level-2 separator
    # every stencil node is owned by exactly one rank (partial interpolation sums are disjoint)
    assert sum(r[2] for r in res) == res[0][3]
    # local-slab I/O (kfbi_local_slab): each rank's f/u box is its slab's grid columns, all j; the boxes
    # tile the unknown columns 1..N−1, and the workspace of a rank holds its slab's spectra only
    for r, sl in zip(res, slabs):
        assert r[4] == (sl["col_lo"], 0) and r[5] == (sl["col_hi"] - sl["col_lo"] + 1, n + 1)
    assert sum(r[5][0] for r in res) == n - 1
    assert all(r[6] < 0.75 * r[7] for r in res)


def _worker3(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2404_15249_b200 import KFBI, broadcast_unique_id
        nid = broadcast_unique_id()
        k = KFBI(W.C4(64), workspace=False, world=world, rank=rank, nccl_id=nid)
        sl = k.slab()
        planes = k.setup_dump(2).reshape(-1, 3)[:, 0]            # x-planes of all stencil nodes
        owned = int(((planes >= sl["i_lo"]) & (planes <= sl["i_hi"])).sum())
        out = [None] * world
        k1 = KFBI(W.C4(64), workspace=False)
        dist.all_gather_object(out, (sl, owned, int(planes.size), k.local_offset, k.local_shape,
                                     k.workspace_bytes, k1.workspace_bytes))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_slab_partition_3d(world):
    """3D slabs are whole ADM blocks of x-planes; plane and stencil-row ranges tile disjointly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker3, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    slabs = [r[0] for r in res]
    n = 64
    assert slabs[0]["b_lo"] == 0 and slabs[-1]["b_hi"] == n // 16
    assert slabs[0]["i_lo"] == 1 and slabs[-1]["i_hi"] == n - 1 and slabs[0]["w_lo"] == 0
    for a, b in zip(slabs[:-1], slabs[1:]):
        assert a["b_hi"] == b["b_lo"] and a["i_hi"] + 1 == b["i_lo"] and a["w_hi"] == b["w_lo"]
        assert a["b_hi"] * 16 == a["i_hi"]                            # slab ends on a block separator
    assert sum(r[1] for r in res) == res[0][2]                        # stencil nodes owned once
    for r, sl in zip(res, slabs):   # local-slab I/O boxes = the slab's x-planes (all j, k)
        assert r[3] == (sl["i_lo"], 0, 0) and r[4] == (sl["i_hi"] - sl["i_lo"] + 1, n + 1, n + 1)
    assert sum(r[4][0] for r in res) == n - 1
    # the two (N−1)·N² working arrays shrink to the slab's planes (≤ 20 N² doubles of level-2 tables added)
    assert all(r[5] <= r[6] - 2 * (n - 1 - r[4][0]) * n * n * 8 + 20 * n * n * 8 for r in res)
