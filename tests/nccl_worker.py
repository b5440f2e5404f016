"""Multi-process (one GPU per rank, NCCL over NVLink) parity worker.

Run by tests/test_nccl_gpu.py as
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tests/nccl_worker.py
Every rank builds the same seeded inputs, puts only the blocks it owns, runs
the distributed drivers through the C-ABI (NCCL transport), gathers its C
blocks to rank 0 over gloo, and rank 0 checks them against the oracle
(pattern bit-exact, values <= 1e-12 Frobenius).  Exits non-zero on mismatch.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from helpers import assert_parity  # noqa: E402
from oracle.oracle import Blocks, Oracle  # noqa: E402
from paper_1910_13555_b200 import dist as d  # noqa: E402
from paper_1910_13555_b200.store import Context, unique_id  # noqa: E402


def owned(blocks: Blocks, m):
    """the blocks of `blocks` this process owns under m's layout"""
    keep = [t for t in range(blocks.nblk) if m.owner_rank(int(blocks.bi[t]), int(blocks.bj[t]))
            in m.comm.local_ranks()]
    off = blocks.offsets()
    vals = np.concatenate([blocks.vals[off[t]:off[t + 1]] for t in keep]) if keep else np.zeros(0)
    return blocks.bi[keep], blocks.bj[keep], vals


def build(blocks, grid, comm):
    m = d.new_matrix_round_robin(d.Blocking(blocks.rsz), d.Blocking(blocks.csz), grid, comm)
    bi, bj, v = owned(blocks, m)
    if len(bi):
        m.put_blocks(bi, bj, v)
    return m


def gather_c(c):
    bi, bj, v = c.blocks()
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, (bi, bj, v))
    if dist.get_rank() != 0:
        return None
    bi = np.concatenate([p[0] for p in parts])
    bj = np.concatenate([p[1] for p in parts])
    rs, cs = c.rows().sizes(), c.cols().sizes()
    sizes = [rs[i] * cs[j] for p in parts for i, j in zip(p[0], p[1])]
    vals_list = []
    for p in parts:
        off = 0
        for i, j in zip(p[0], p[1]):
            n = rs[i] * cs[j]
            vals_list.append(p[2][off:off + n])
            off += n
    order = np.lexsort((bj, bi))
    vals = np.concatenate([vals_list[t] for t in order]) if len(order) else np.zeros(0)
    del sizes
    return Blocks(rs, cs, bi[order], bj[order], vals)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = Context(local, world, rank, obj[0])
    comm = d.SimComm.nccl(ctx)
    o = Oracle()
    failures = 0
    q = int(round(world ** 0.5))
    cases = []
    if q * q == world:
        cases.append(("cannon", q))
    cases += [("case1", 1), ("case2", 1), ("case2g", 1)]
    # the B gather again on the same communicator: speculative segment
    # capacities (a slightly smaller B fits; a much denser one misses and is
    # redone exactly), then eps > 0 (always exact)
    cases += [("case2g-spec", 1, 21, 0.40), ("case2g-miss", 1, 31, 0.85),
              ("case2g-spec2", 1, 41, 0.80)]
    rs = np.array([5, 13, 23, 7, 13, 5, 23, 11, 9, 17, 4, 23], np.int32)
    ks = np.array([13, 5, 23, 8, 16, 23, 5, 13], np.int32)
    ns = np.array([23, 7, 5, 13, 20, 9, 23], np.int32)
    for case in cases:
        algo, gq = case[0], case[1]
        seed, occ = (case[2], case[3]) if len(case) > 2 else (11, 0.45)
        A = o.random_matrix(seed, rs, ks, occ)
        B = o.random_matrix(seed + 1, ks, ns, occ)
        Cin = o.random_matrix(seed + 2, rs, ns, 0.2)
        grid = d.ProcessGrid([gq, gq])
        a, b, c = build(A, grid, comm), build(B, grid, comm), build(Cin, grid, comm)
        if algo == "cannon":
            st = d.multiply_cannon(comm, a, b, c)
        elif algo == "case1":
            st = d.multiply_reduce_case1(comm, a, b, c, world)
        else:
            st = d.multiply_virtual_case2(comm, a, b, c, world, gather=algo.startswith("case2g"))
        got = gather_c(c)
        if rank == 0:
            want, _, _ = o.multiply(A, B, Cin)
            try:
                err = assert_parity(got, want)
                print(f"[nccl world={world}] {algo}: OK rel_err={err:.2e} "
                      f"sent={st['elements_sent']}", flush=True)
            except AssertionError as e:
                failures += 1
                print(f"[nccl world={world}] {algo}: FAIL {e}", flush=True)
    # distributed tensor contraction with remaps: rank 3 over
    # two indices and rank 4, against einsum of the dense operands
    import itertools
    from paper_1910_13555_b200.tensor import DistTensor, contract_dist
    tgrid = d.ProcessGrid([q, q]) if q * q == world else d.ProcessGrid([world, 1])
    rng = np.random.default_rng(5)

    def items(sizes, occ):
        out = []
        for coords in itertools.product(*[range(len(z)) for z in sizes]):
            if rng.random() < occ:
                out.append((list(coords), rng.standard_normal([int(z[c]) for z, c in
                                                               zip(sizes, coords)])))
        return out

    def dense(sizes, its):
        offs = [np.concatenate([[0], np.cumsum(z)]) for z in sizes]
        out = np.zeros([int(o[-1]) for o in offs])
        for coords, blk in its:
            out[tuple(slice(offs[k][c], offs[k][c] + blk.shape[k])
                      for k, c in enumerate(coords))] = blk
        return out

    s3 = [np.array([2, 3, 2], np.int32), np.array([4, 2], np.int32), np.array([3, 1, 2], np.int32)]
    s4 = [np.array([3, 5], np.int32), np.array([4, 2], np.int32), np.array([2, 6], np.int32),
          np.array([5, 1], np.int32)]
    for name, sa, sb, amap, bmap, ca, cb, sc, cmap, spec in (
            ("tensor3", s3, [s3[1], s3[2], s3[0]], ([2], [0, 1]), ([0, 1], [2]), [1, 2], [0, 1],
             [s3[0], s3[0]], ([1], [0]), "mkl,kln->mn"),
            ("tensor4", s4, [s4[3], s4[1], s4[2], s4[0]], ([0, 2], [1, 3]), ([1], [0, 2, 3]),
             [1, 3], [1, 0], [s4[0], s4[2], s4[2], s4[0]], ([0, 3], [1, 2]), "ikjl,lkmn->ijmn")):
        ia, ib = items(sa, 0.6), items(sb, 0.6)
        A = DistTensor(comm, sa, *amap, grid=tgrid)
        A.put_blocks(ia)
        B = DistTensor(comm, sb, *bmap, grid=tgrid)
        B.put_blocks(ib)
        Cm = DistTensor(comm, sc, *cmap, grid=tgrid)
        comm.reset_ledger()
        contract_dist(A, B, ca, cb, Cm)
        local = torch.from_numpy(Cm.to_dense())
        dist.all_reduce(local)   # every block lives on exactly one rank
        remap_sent = torch.tensor([float(comm.ledger().rank_phase(rank, "tensor_remap")
                                         .elements_sent)])
        dist.all_reduce(remap_sent)
        if rank == 0:
            want = np.einsum(spec, dense(sa, ia), dense(sb, ib))
            err = float(np.sqrt(np.sum((local.numpy() - want) ** 2) / np.sum(want ** 2)))
            ok = err <= 1e-12 and remap_sent.item() > 0
            failures += 0 if ok else 1
            print(f"[nccl world={world}] {name}: {'OK' if ok else 'FAIL'} rel_err={err:.2e} "
                  f"remap_sent={int(remap_sent.item())}", flush=True)
    flag = torch.tensor([failures])
    dist.broadcast(flag, 0)
    comm.close()
    ctx.close()
    dist.destroy_process_group()
    sys.exit(1 if int(flag.item()) else 0)


if __name__ == "__main__":
    main()
