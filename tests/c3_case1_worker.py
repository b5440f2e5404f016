"""BASELINE config 3 through multiply_reduce_case1 on P GPUs (one process per GPU,
NCCL), checked against the oracle -- not against a 1-GPU run of this library.

Run by tests/test_nccl_gpu.py::test_c3_case1_vs_oracle as
    torchrun --nproc-per-node P tests/c3_case1_worker.py [--occ 0.1]
C (2000 x 2000) += A (2000 x 400 000) * B (400 000 x 2000), blocks of 20
(multiply_rect.hpp:123-192).  Every rank owns the K-slab of A and B that case 1
multiplies locally; the partial C blocks are reduced to their owners over
NVLink.  Rank 0 gathers C over gloo and compares with the oracle's C for the
full A and B (pattern bit-exact, values <= 1e-12 Frobenius-relative, globally
and per block).  Exits non-zero on mismatch.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from helpers import assert_parity  # noqa: E402
from oracle.oracle import Blocks, Oracle  # noqa: E402
from run_c3_dist import BS, KB, MB, NB, slab  # noqa: E402  (seeded input generator)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--occ", type=float, default=0.10)
    args = ap.parse_args()
    from paper_1910_13555_b200 import dist as dd
    from paper_1910_13555_b200.store import Context, unique_id
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    obj = [unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    ctx = Context(local, world, rank, obj[0])
    comm = dd.SimComm.nccl(ctx)
    m_sz, k_sz, n_sz = (np.full(n, BS, np.int32) for n in (MB, KB, NB))
    ks = (np.arange(KB) * world) // KB
    k0, k1 = int(np.searchsorted(ks, rank)), int(np.searchsorted(ks, rank + 1))
    A = slab("a", k0, k1, args.occ)
    B = slab("b", k0, k1, args.occ)
    a = dd.new_matrix(dd.Blocking(m_sz), dd.Blocking(k_sz), dd.ProcessGrid([1, world]),
                      np.zeros(MB, np.int64), ks, comm)
    b = dd.new_matrix(dd.Blocking(k_sz), dd.Blocking(n_sz), dd.ProcessGrid([world, 1]), ks,
                      np.zeros(NB, np.int64), comm)
    a.local(rank).put_blocks(*A)
    b.local(rank).put_blocks(*B)
    c = dd.new_matrix(dd.Blocking(m_sz), dd.Blocking(n_sz), dd.ProcessGrid([world, 1]),
                      np.arange(MB) % world, np.zeros(NB, np.int64), comm)
    st = None
    for _ in range(2):   # second call: steady-state buffers
        c.local(rank).clear()
        st = dd.multiply_reduce_case1(comm, a, b, c, world)
    bi, bj, v = c.local(rank).export()
    parts = [None] * world
    dist.all_gather_object(parts, (bi, bj, v))
    fl = torch.tensor([st["flops"]], dtype=torch.float64)
    dist.all_reduce(fl)
    ok = 1
    if rank == 0:
        gi = np.concatenate([p[0] for p in parts])
        gj = np.concatenate([p[1] for p in parts])
        gv = np.concatenate([p[2] for p in parts]).reshape(-1, BS * BS)
        order = np.lexsort((gj, gi))
        got = Blocks(m_sz, n_sz, gi[order], gj[order], gv[order].ravel())
        fa = Blocks(m_sz, k_sz, *slab("a", 0, KB, args.occ))
        fb = Blocks(k_sz, n_sz, *slab("b", 0, KB, args.occ))
        want, _, oflops = Oracle().multiply(fa, fb, Blocks.empty(m_sz, n_sz))
        try:
            assert abs(fl.item() - oflops) <= 1e-9 * oflops, (fl.item(), oflops)
            err = assert_parity(got, want)
            print(f"[c3 case1 world={world} occ={args.occ}] OK blocks={got.nblk} "
                  f"gflop={oflops / 1e9:.2f} rel_err={err:.2e}", flush=True)
        except AssertionError as e:
            ok = 0
            print(f"[c3 case1 world={world}] FAIL {e}", flush=True)
    flag = torch.tensor([ok])
    dist.broadcast(flag, 0)
    comm.close()
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if int(flag.item()) else 1)


if __name__ == "__main__":
    main()
