"""BASELINE config 3 on P GPUs through the CARMA case-1 driver (one process per
GPU, NCCL): C (2000 x 2000) += A (2000 x 400 000) * B (400 000 x 2000), blocks of
20, occupancy 10-50 %.  Strong scaling: every rank owns the K-slab of A
(columns) and B (rows) that case 1 multiplies locally (multiply_rect.hpp:123-192),
so the timed call is the local multiply + the one-hop reduction of the partial
C blocks to their owners over NVLink.

  torchrun --nproc-per-node P tools/run_c3_dist.py [--occ 0.1] [--steps 3] [--check]

Inputs: numpy PCG64 seeded per K-slab (independent of P).  --check: rank 0
recomputes C on its own GPU from the full A and B (single-GPU multiply) and
compares (pattern bit-exact, values <= 1e-12 Frobenius-relative).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MB, KB, NB, BS = 100, 20000, 100, 20   # block rows of A/C, K blocks, block cols of B/C, size
KCHUNK = 500                            # generation granularity along K (seeding unit)


def slab(kind, k0, k1, occ):
    """(bi, bj, vals) of A[:, k0:k1] (kind 'a') or B[k0:k1, :] (kind 'b'), global
    block indices, canonical order, seeded per KCHUNK of K."""
    bis, bjs, vs = [], [], []
    for c0 in range(k0 - k0 % KCHUNK, k1, KCHUNK):
        g = np.random.default_rng([1 if kind == "a" else 2, c0])
        if kind == "a":
            mask = g.random((MB, KCHUNK)) < occ
        else:
            mask = g.random((KCHUNK, NB)) < occ
        bi, bj = np.nonzero(mask)
        vals = g.standard_normal(len(bi) * BS * BS)
        if kind == "a":
            bj = bj + c0
            keep = (bj >= k0) & (bj < k1)
        else:
            bi = bi + c0
            keep = (bi >= k0) & (bi < k1)
        idx = np.nonzero(keep)[0]
        bis.append(bi[idx])
        bjs.append(bj[idx])
        vs.append(vals.reshape(-1, BS * BS)[idx].ravel())
    bi, bj, v = np.concatenate(bis), np.concatenate(bjs), np.concatenate(vs)
    order = np.lexsort((bj, bi))
    return (bi[order].astype(np.int64), bj[order].astype(np.int64),
            v.reshape(-1, BS * BS)[order].ravel())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--occ", type=float, default=0.10)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    args = ap.parse_args()
    from paper_1910_13555_b200 import dist as dd
    from paper_1910_13555_b200.store import Context, LocalStore, multiply_local, unique_id
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = Context(local, world, rank, obj[0]) if world > 1 else Context(local)
    comm = dd.SimComm.nccl(ctx) if world > 1 else dd.SimComm(dd.ProcessGrid([1]), ctx=ctx)
    m_sz, k_sz, n_sz = (np.full(n, BS, np.int32) for n in (MB, KB, NB))
    ks = (np.arange(KB) * world) // KB           # ChunkPartition-like K-slab owner
    k0 = int(np.searchsorted(ks, rank)), int(np.searchsorted(ks, rank + 1))
    t0 = time.time()
    A = slab("a", k0[0], k0[1], args.occ)
    B = slab("b", k0[0], k0[1], args.occ)
    gen_s = time.time() - t0
    # case-1 layouts: A on a 1 x P grid by K columns, B on P x 1 by K rows
    a = dd.new_matrix(dd.Blocking(m_sz), dd.Blocking(k_sz), dd.ProcessGrid([1, world]),
                      np.zeros(MB, np.int64), ks, comm)
    b = dd.new_matrix(dd.Blocking(k_sz), dd.Blocking(n_sz), dd.ProcessGrid([world, 1]), ks,
                      np.zeros(NB, np.int64), comm)
    a.local(rank).put_blocks(*A)
    b.local(rank).put_blocks(*B)
    c = dd.new_matrix(dd.Blocking(m_sz), dd.Blocking(n_sz), dd.ProcessGrid([world, 1]),
                      np.arange(MB) % world, np.zeros(NB, np.int64), comm)
    stream = torch.cuda.ExternalStream(ctx.stream)
    times, st = [], None
    for it in range(1 + args.steps):
        c.local(rank).clear()
        ctx.sync()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
        st = dd.multiply_reduce_case1(comm, a, b, c, world)
        with torch.cuda.stream(stream):
            e1.record(stream)
        torch.cuda.synchronize()
        if it >= 1:
            times.append(e0.elapsed_time(e1))
    ms = torch.tensor([float(np.median(times))], dtype=torch.float64)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    fl = torch.tensor([st["flops"]], dtype=torch.float64)
    dist.all_reduce(fl)
    out = {"config": "c3", "workload": f"C 2000x2000 += A 2000x400000 * B 400000x2000, bs 20, "
                                      f"occ {args.occ:.2f}", "gpus": world,
           "algorithm": "multiply_reduce_case1 (K slabs, one-hop NVLink reduction)",
           "ms_median_max_over_ranks": round(float(ms.item()), 4),
           "useful_gflop": round(float(fl.item()) / 1e9, 3),
           "tflops_total": round(float(fl.item()) / (float(ms.item()) * 1e-3) / 1e12, 3),
           "gen_s": round(gen_s, 1)}
    if args.check:
        bi, bj, v = c.local(rank).export()
        parts = [None] * world
        dist.all_gather_object(parts, (bi, bj, v))
        if rank == 0:
            from paper_1910_13555_b200.store import LocalStore as LS
            fa = slab("a", 0, KB, args.occ)
            fb = slab("b", 0, KB, args.occ)
            one = Context(local)
            sa, sb, sc = LS(one, m_sz, k_sz), LS(one, k_sz, n_sz), LS(one, m_sz, n_sz)
            sa.put_blocks(*fa)
            sb.put_blocks(*fb)
            multiply_local(one, sa, sb, sc)
            wi, wj, wv = sc.export()
            gi = np.concatenate([p[0] for p in parts])
            gj = np.concatenate([p[1] for p in parts])
            gv = np.concatenate([p[2] for p in parts])
            order = np.lexsort((gj, gi))
            gv = gv.reshape(-1, BS * BS)[order].ravel()
            assert np.array_equal(gi[order], wi) and np.array_equal(gj[order], wj), "pattern"
            err = float(np.linalg.norm(gv - wv) / np.linalg.norm(wv))
            assert err <= 1e-12, err
            out["check"] = f"pattern bit-exact, frobenius rel err {err:.2e} vs 1-GPU multiply"
    if rank == 0:
        print(json.dumps(out), flush=True)
    comm.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
