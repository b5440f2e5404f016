"""The N>1 host path on CPU: world_size-2 gloo processes run the bench's
per-rank input slicing and the layout/ownership math of the distributed
drivers, and check the ranks agree (no GPU; the device path is covered by
test_nccl_gpu.py on real GPUs)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1910_13555_b200 import dist as d
    try:
        nb = 40
        # bench slicing: A rows of this rank's slab, B rows of its K slab
        abi, abj, _ = bench.make_blocks(bench.SEED_A, nb, nb, 3, 0.2, row0=nb * rank)
        chunk = -(-nb // world)
        part = d.ChunkPartition(nb, world)
        assert (part.begin(rank), part.end(rank)) == (min(nb, chunk * rank),
                                                      min(nb, chunk * (rank + 1)))
        gathered = [None] * world
        dist.all_gather_object(gathered, (abi + nb * rank, abj))
        # A slabs: disjoint rows, rank r owns [nb r, nb r + nb)
        for r, (bi, _) in enumerate(gathered):
            assert bi.min() >= nb * r and bi.max() < nb * (r + 1)
        # the slab layout's owner of every block is the rank holding it
        grid = d.ProcessGrid([world, 1])
        rdist = np.arange(nb * world) // nb
        for r, (bi, bj) in enumerate(gathered):
            owners = {grid.rank_of([int(rdist[i]), 0]) for i in bi}
            assert owners == {r}
        # Cannon neighbours agree across ranks on a 1 x world ring of grids
        qg = d.ProcessGrid([1, world])
        left = qg.rank_of([0, (rank - 1) % world])
        right = qg.rank_of([0, (rank + 1) % world])
        nbrs = [None] * world
        dist.all_gather_object(nbrs, (left, right))
        for r, (lft, _) in enumerate(nbrs):
            assert nbrs[lft][1] == r
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_host_path():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(2))
    assert res == {0: "ok", 1: "ok"}, res
