"""Measured time of every distributed algorithm on P GPUs (one process per
GPU, NCCL), the data the NVLink-aware selection model is fitted to
(dist.predicted_time_b200):

  torchrun --nproc-per-node P tools/algo_sweep.py [--out file.jsonl]

Workloads (synthetic, seeded): square (c1 shape), tall-skinny (c3, 10 %),
dense-ish (c5 shape scaled to 512^2 blocks of 32, occ 0.5) and wide-C (C much
larger than A and B).  Inputs in one neutral layout -- round robin on the
most square 2-D grid of P ranks -- for every algorithm: Cannon (square P only)
multiplies in place, case 1 / case 2 redistribute as the reference does
(multiply_rect.hpp:123-238), so each time includes its own data movement.
CUDA events around the driver call, max over ranks, median of 3 after a
warm-up.  One JSON line per (workload, algorithm) on rank 0."""
import argparse
import json
import math
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def workloads():
    rng = np.random.default_rng
    yield "square", (np.full(400, 23), np.full(400, 23), np.full(400, 23), 0.10, 0.10)
    yield "tall_skinny", (np.full(100, 20), np.full(20000, 20), np.full(100, 20), 0.10, 0.10)
    yield "dense", (np.full(512, 32), np.full(512, 32), np.full(512, 32), 0.5, 0.5)
    yield "wide_c", (np.full(1500, 13), np.full(60, 13), np.full(1500, 13), 0.3, 0.3)
    del rng


def blocks(seed, rsz, csz, occ, own):
    g = np.random.default_rng(seed)
    mask = g.random((len(rsz), len(csz))) < occ
    bi, bj = np.nonzero(mask)
    sizes = rsz[bi].astype(np.int64) * csz[bj]
    keep = own(bi, bj)
    vals = g.standard_normal(int(sizes.sum()))
    off = np.concatenate([[0], np.cumsum(sizes)])
    sel = np.nonzero(keep)[0]
    v = np.concatenate([vals[off[t]:off[t + 1]] for t in sel]) if len(sel) else np.zeros(0)
    return bi[sel].astype(np.int64), bj[sel].astype(np.int64), v, int(mask.sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    from paper_1910_13555_b200 import dist as dd
    from paper_1910_13555_b200.store import Context, unique_id
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = Context(local, world, rank, obj[0]) if world > 1 else Context(local)
    comm = dd.SimComm.nccl(ctx) if world > 1 else dd.SimComm(dd.ProcessGrid([1]), ctx=ctx)
    q = int(round(math.sqrt(world)))
    gr = [q, q] if q * q == world else [world, 1]
    grid = dd.ProcessGrid(gr)
    stream = torch.cuda.ExternalStream(ctx.stream)
    out = open(args.out, "a") if (args.out and rank == 0) else None
    for name, (ms, ks, ns, oa, ob) in workloads():
        if args.only and name != args.only:
            continue
        ms, ks, ns = (np.asarray(x, np.int32) for x in (ms, ks, ns))
        B_ = dd.Blocking
        mats, occs = [], []
        for seed, rs, cs, occ in ((11, ms, ks, oa), (12, ks, ns, ob)):
            m = dd.new_matrix_round_robin(B_(rs), B_(cs), grid, comm)
            # round robin owner: grid coords (i mod gr0, j mod gr1), row-major rank
            own = lambda bi, bj: (bi % gr[0]) * gr[1] + (bj % gr[1]) == rank  # noqa: E731
            bi, bj, v, ntot = blocks(seed, rs, cs, occ, own)
            if len(bi):
                m.local(rank).put_blocks(bi, bj, v)
            mats.append(m)
            occs.append(ntot / float(len(rs) * len(cs)))
        a, b = mats
        algos = (["cannon"] if q * q == world else []) + ["case1", "case2"]
        for algo in algos:
            ts, st = [], None
            for it in range(4):
                c = dd.new_matrix_round_robin(B_(ms), B_(ns), grid, comm)
                ctx.sync()
                dist.barrier()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(stream):
                    e0.record(stream)
                if algo == "cannon":
                    st = dd.multiply_cannon(comm, a, b, c)
                elif algo == "case1":
                    st = dd.multiply_reduce_case1(comm, a, b, c, world)
                else:
                    st = dd.multiply_virtual_case2(comm, a, b, c, world, gather=True)
                with torch.cuda.stream(stream):
                    e1.record(stream)
                ctx.sync()
                torch.cuda.synchronize()
                if it:
                    ts.append(e0.elapsed_time(e1))
                c._close()
            t = torch.tensor([float(np.median(ts))], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            fl = torch.tensor([st["flops"]], dtype=torch.float64)
            dist.all_reduce(fl)
            if rank == 0:
                line = {"workload": name, "algo": algo, "gpus": world, "grid": gr,
                        "ms": round(float(t.item()), 4), "gflop": round(float(fl.item()) / 1e9, 3),
                        "m": int(ms.sum()), "n": int(ns.sum()), "k": int(ks.sum()),
                        "occ_a": round(occs[0], 6), "occ_b": round(occs[1], 6)}
                print(json.dumps(line), flush=True)
                if out:
                    out.write(json.dumps(line) + "\n")
        for m in mats:
            m._close()
    comm.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
