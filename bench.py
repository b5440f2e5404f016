#!/usr/bin/env python3
"""bench.py -- block-sparse FP64 useful GFLOP/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[0], the config the metric is quoted on:
"10% occupancy with 23x23 blocks"): C += A*B with A, B 400 x 400 blocks of
23 x 23 (N = 9,200), 10 % random block occupancy, C_in empty, eps = 0.
Synthetic inputs: block presence Bernoulli(0.10), values N(0,1), seeded
(A: 1001, B: 1002) with numpy's PCG64 so both arms regenerate identical inputs.

A "step" = one full multiply call (stack generation, symbolic C pattern,
small-GEMM numeric phase, C install).  N > 1 (torchrun, one process per GPU):
weak scaling over a row-slab distribution -- every rank owns 400 block-rows of
A and C (a 400*N x 400 A), B (400 x 400 blocks) is K-sliced across ranks and
circulates over NCCL in a ring (the reference's multiply_virtual_case2
schedule, multiply_rect.hpp:199-238), so per-rank work equals the N = 1 step.

Impls:
  (default)          the B200 product through its C-ABI (libbtcuda.so)
  --impl reference   the reference's own CPU path (oracle/_ref, compiled from the
                     unmodified /root/reference headers) on the box's host cores
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NB, BS, OCC = 400, 23, 0.10
SEED_A, SEED_B = 1001, 1002
FP64_PEAK_TFLOPS = 37.1   # measured: tools/microbench/fp64_peak.cu on B200 (profiles/)
# dram__bytes_read.sum + dram__bytes_write.sum of one k_smm_dmma launch on this
# workload, from `ncu --set full` of this bench (profiles/r02/ncu_bench_dmma_summary.txt):
# 0.646 GB read + 0.697 GB written (algorithmic: 0.80 GB)
NCU_TRAFFIC_BYTES = 1.3422e9


METRIC = "block-sparse FP64 useful GFLOP/s"
DATA = "synthetic (seeded Bernoulli(0.10) block presence, N(0,1) values)"


L2_NOTE = ("GPU arm: L2 flushed (256 MB write) before every timed step; "
           "CPU reference arm: no flush (host caches hold nothing across a 15 GFLOP step)")


def bench_config(world, products_per_rank, flops_per_rank):
    """The `config` object, IDENTICAL in both arms (the workload; how each arm
    runs it is in the line's top-level `distribution`)."""
    return {
        "workload": "c1: 400x400 blocks of 23x23 (N=9200) per rank, occ 0.10, C_in empty, eps 0",
        "products_per_rank": int(products_per_rank),
        "useful_gflop_per_rank": round(flops_per_rank / 1e9, 4),
        "l2": L2_NOTE,
    }


# --------------------------------------------------------------- inputs
def make_blocks(seed: int, nbr: int, nbc: int, bs: int, occ: float, row0: int = 0):
    """Canonical (bi, bj, vals) block list, Bernoulli(occ) presence, N(0,1) values.
    Rows [row0, row0+nbr) of a conceptually larger matrix (row-sliced seeding keeps
    every rank's slab independent of the world size)."""
    bis, bjs, vs = [], [], []
    for r in range(row0, row0 + nbr):
        g = np.random.default_rng([seed, r])
        mask = g.random(nbc) < occ
        js = np.nonzero(mask)[0].astype(np.int64)
        bis.append(np.full(len(js), r - row0, np.int64))
        bjs.append(js)
        vs.append(g.standard_normal(len(js) * bs * bs))
    return np.concatenate(bis), np.concatenate(bjs), np.concatenate(vs)


def useful_flops_host(a_bi, a_bj, b_bi, b_bj, bs):
    """2*m*n*k per (i,k,j) with A_ik and B_kj stored."""
    b_rows = np.bincount(b_bi, minlength=NB)
    return 2.0 * bs ** 3 * float(b_rows[a_bj].sum())


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        if os.environ.get("BT_BENCH_NO_SMI"):  # diagnosis only: no sampler
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.25)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# --------------------------------------------------------------- reference
def run_reference(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref/libbtref.so) on this box's
    host cores: multiply_cannon on the largest square grid <= nproc (one
    std::thread per simulated rank, comm.hpp:273-290)."""
    if rank != 0:
        return None
    from oracle.oracle import Blocks, Reference  # the one place bench runs oracle/
    ref = Reference()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    q = int(np.floor(np.sqrt(cores or 1)))
    sz = np.full(NB, BS, np.int32)
    abi, abj, av = make_blocks(SEED_A, NB, NB, BS, OCC)
    bbi, bbj, bv = make_blocks(SEED_B, NB, NB, BS, OCC)
    A = Blocks(sz, sz, abi, abj, av)
    B = Blocks(sz, sz, bbi, bbj, bv)
    C = Blocks.empty(sz, sz)
    flops = useful_flops_host(abi, abj, bbi, bbj, BS)
    nprod = flops / (2.0 * BS ** 3)
    for _ in range(args.warmup):
        ref.multiply(A, B, C, "cannon", q, q * q)
    times = []
    for _ in range(args.steps):
        _, secs, _ = ref.multiply(A, B, C, "cannon", q, q * q)
        times.append(secs)
    t = float(np.sum(times))
    val = flops * args.steps / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC,
        "value": round(val, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA,
        "config": bench_config(world, int(round(nprod)), flops),
        "distribution": (f"reference multiply_cannon on a {q}x{q} simulated grid ({q * q} host "
                         f"threads); each step is one c1 instance (rank 0's slab of the "
                         f"{world}-rank job)"),
        "cpu_baseline": {"value": round(val, 3), "unit": "GFLOP/s", "cores": q * q,
                         "kind": "reference",
                         "sample": f"full c1 instance per step ({flops/1e9:.2f} GFLOP)"},
        "e2e": {"value": round(val, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return line


def cpu_baseline_sample(reps: int = 3):
    """cpu_baseline for the product line: the reference on ONE core (1x1 Cannon),
    `reps` full c1 instances (~3 s each on this pool's hosts, ~10 s in all)."""
    from oracle.oracle import Blocks, Reference
    ref = Reference()
    sz = np.full(NB, BS, np.int32)
    abi, abj, av = make_blocks(SEED_A, NB, NB, BS, OCC)
    bbi, bbj, bv = make_blocks(SEED_B, NB, NB, BS, OCC)
    flops = useful_flops_host(abi, abj, bbi, bbj, BS)
    A, B = Blocks(sz, sz, abi, abj, av), Blocks(sz, sz, bbi, bbj, bv)
    secs, out = 0.0, None
    for _ in range(reps):
        out, t, _ = ref.multiply(A, B, Blocks.empty(sz, sz), "cannon", 1, 1)
        secs += t
    return {"value": round(reps * flops / secs / 1e9, 3), "unit": "GFLOP/s", "cores": 1,
            "kind": "reference",
            "sample": f"{reps} full c1 instances, reference multiply_cannon on a 1x1 grid "
                      f"({reps * flops / 1e9:.2f} GFLOP in {secs:.2f} s)"}, out


# --------------------------------------------------------------- product
def relaunch_under_torchrun(n: int):
    """`bench.py --gpus N` without a launcher: re-exec as N ranks (one process per
    GPU) under torch.distributed.run on 127.0.0.1, NCCL's init lines visible."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    if env.get("NCCL_DEBUG", "").upper() not in ("INFO", "TRACE"):
        env["NCCL_DEBUG"] = "INFO"          # the communicator init lines (ranks, NVLink)
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        # to stderr: stdout's last line stays the JSON line (NCCL's teardown
        # messages of the other ranks would otherwise follow it)
        env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execvpe(sys.executable, cmd, env)


def parity_vs_reference(c_store, ref_c):
    """The bench's own GPU C (rank 0's slab) against the reference's C for the same
    inputs: pattern bit-exact, per-block and global Frobenius-relative error
    (oracles.hpp:49-57; north_star bar 1e-12)."""
    bi, bj, v = c_store.export()
    exact = bool(len(bi) == ref_c.nblk and np.array_equal(bi, ref_c.bi)
                 and np.array_equal(bj, ref_c.bj) and v.shape == ref_c.vals.shape)
    out = {"pattern_exact": exact, "blocks": int(len(bi)),
           "checked": "rank 0's C vs the reference multiply_cannon (1x1) on the same inputs"}
    if exact:
        d = (v - ref_c.vals) ** 2
        r = ref_c.vals ** 2
        off = ref_c.offsets()[:-1]
        per = np.sqrt(np.add.reduceat(d, off) / np.maximum(np.add.reduceat(r, off), 1e-300))
        out["max_frob"] = float(per.max()) if len(per) else 0.0
        out["global_frob"] = float(np.sqrt(d.sum() / r.sum())) if r.sum() > 0 else 0.0
        out["ok"] = out["max_frob"] <= 1e-12
    else:
        out["ok"] = False
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="N > 1: skip rank 0's check against the reference")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        relaunch_under_torchrun(args.gpus)   # does not return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "b200" and world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1910_13555_b200.store import Context, LocalStore, multiply_local, unique_id
    from paper_1910_13555_b200 import dist as dd

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
        obj = [unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = Context(local, world, rank, obj[0])
    else:
        ctx = Context(local)
    # events around the multiply kernels without a wait inside the call; the
    # numeric kernel's device time is read after each timed step (outside e0..e1)
    ctx.set_timing(2)
    stream = torch.cuda.ExternalStream(ctx.stream)
    sz = np.full(NB, BS, np.int32)

    # ---- inputs (host, pinned): A/C row slab of this rank, B K-slab of this rank
    abi, abj, av = make_blocks(SEED_A, NB, NB, BS, OCC, row0=NB * rank)
    chunk = -(-NB // world)   # ChunkPartition (partition.hpp:17-41) of B's block rows
    k0, k1 = min(NB, chunk * rank), min(NB, chunk * (rank + 1))
    bbi_all, bbj_all, bv_all = make_blocks(SEED_B, NB, NB, BS, OCC)
    sel = (bbi_all >= k0) & (bbi_all < k1)
    bsize = BS * BS
    bbi, bbj = bbi_all[sel], bbj_all[sel]
    bv = np.ascontiguousarray(bv_all.reshape(-1, bsize)[np.nonzero(sel)[0]].ravel())
    av_pin = torch.from_numpy(av).pin_memory()
    bv_pin = torch.from_numpy(bv).pin_memory()
    flops_rank = useful_flops_host(abi, abj, bbi_all, bbj_all, BS)

    if world == 1:
        a = LocalStore(ctx, sz, sz)
        a.put_blocks(abi, abj, av_pin)
        b = LocalStore(ctx, sz, sz)
        b.put_blocks(bbi, bbj, bv_pin)
        c = LocalStore(ctx, sz, sz)

        def step(cc):
            cc.clear()
            return multiply_local(ctx, a, b, cc)
    else:
        # weak scaling: A and C are 400*world x 400 block matrices in row slabs
        # (rank r owns block rows [400 r, 400 r + 400)), B is 400 x 400 in K slabs;
        # the layouts already match case 2's, so a step is the B gather over
        # NVLink + the local multiply (multiply_rect.hpp:199-238)
        comm = dd.SimComm.nccl(ctx)
        grid = dd.ProcessGrid([world, 1])
        rows_a = dd.Blocking.uniform(NB * world, BS)
        cols = dd.Blocking.uniform(NB, BS)
        a = dd.new_matrix(rows_a, cols, grid, np.arange(NB * world) // NB,
                          np.zeros(NB, np.int64), comm)
        a.put_blocks(abi + NB * rank, abj, av)
        b = dd.new_matrix(cols, cols, grid, np.arange(NB) // chunk, np.zeros(NB, np.int64), comm)
        b.put_blocks(bbi, bbj, bv)
        c = dd.new_matrix(rows_a, cols, grid, np.arange(NB * world) // NB,
                          np.zeros(NB, np.int64), comm)

        def step(cc):
            cc.local(rank).clear()
            st = dd.multiply_virtual_case2(comm, a, b, cc, world, gather=True)
            return st

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    # the clock sampler starts BEFORE the warm-up: its start-up pause idles the
    # GPU, so the warm-up steps bring the clocks back up before the timed steps
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    ms_numeric = []
    stats = []
    gc.disable()   # no collector pauses between the host-synchronous API calls
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            with torch.cuda.stream(stream):
                flush.zero_()
            st = step(c)
        ctx.sync()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        k_before = ctx.kernel_count
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()                       # L2 flush, outside the timed events
                ev[s][0].record(stream)
            st = step(c)
            with torch.cuda.stream(stream):
                ev[s][1].record(stream)
            ms_numeric.append(ctx.last_timing()[0])
            stats.append(st)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    kernels = ctx.kernel_count - k_before
    step_ms = [e0.elapsed_time(e1) for e0, e1 in ev]
    if os.environ.get("BT_BENCH_DEBUG"):
        print(f"[rank {rank}] step_ms {np.round(step_ms, 3).tolist()} "
              f"numeric_ms {np.round(ms_numeric, 3).tolist()}", file=sys.stderr, flush=True)
    ms_local = float(np.mean(step_ms))
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops_step = stats[-1]["flops"]
    assert abs(flops_step - flops_rank) <= 1e-6 * flops_rank, (flops_step, flops_rank)
    value = flops_step * world / (ms * 1e-3) / 1e9     # whole-job GFLOP/s

    # ---- dominant kernel roofline (small-GEMM numeric phase, live CUDA events)
    kn_ms = float(np.mean(ms_numeric))
    c_el = c.info()[1] if world == 1 else c.local(rank).info()[1]
    alg_bytes = 8.0 * (av.size + bv.size * world + c_el) + 12.0 * (len(abi) + len(bbi) * world)
    achieved = flops_step / (kn_ms * 1e-3) / 1e12

    # ---- e2e through the public API with host buffers (rank-local).  Every
    # step uploads A and B from pinned host memory (put_blocks), multiplies and
    # reads all of C back (export).  The C read-back is bt_mat_export_async:
    # its D2H runs on a side stream while the next step's uploads and
    # multiply proceed (PCIe is full duplex), so the steady state is bounded
    # by the 667 MB C transfer per step.  Timed over the K steps as a whole,
    # from a synchronised start to the last transfer landing (ctx.sync()).
    couts = [torch.empty(NB * NB * bsize, dtype=torch.float64).pin_memory() for _ in range(2)]
    h2d = av.nbytes + bv.nbytes + 16 * (len(abi) + len(bbi))
    d2h = 0

    if world == 1:   # the user's stores, refilled every step (clear keeps capacity)
        ea, eb, ec = LocalStore(ctx, sz, sz), LocalStore(ctx, sz, sz), LocalStore(ctx, sz, sz)

    def e2e_step(s):
        nonlocal d2h
        if world == 1:
            for x in (ea, eb, ec):
                x.clear()
            ea.put_blocks(abi, abj, av_pin)
            eb.put_blocks(bbi, bbj, bv_pin)
            multiply_local(ctx, ea, eb, ec)
            ci, cj, _ = ec.export(couts[s % 2], asynchronous=True)
            d2h = 8 * int(ec.info()[1]) + 16 * len(ci)
        else:
            a.local(rank).clear()
            b.local(rank).clear()
            c.local(rank).clear()
            a.local(rank).put_blocks(abi + NB * rank, abj, av_pin)
            b.local(rank).put_blocks(bbi, bbj, bv_pin)
            dd.multiply_virtual_case2(comm, a, b, c, world, gather=True)
            ci, cj, _ = c.local(rank).export(couts[s % 2], asynchronous=True)
            d2h = 8 * int(c.local(rank).info()[1]) + 16 * len(ci)

    for s in range(args.warmup):
        e2e_step(s)
    ctx.sync()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for s in range(args.steps):
        e2e_step(s)
    ctx.sync()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world == 1:
        for x in (ea, eb, ec):
            x.close()
    gc.enable()
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = flops_step * world / e2e_s / 1e9

    # ---- parity of this run's own C (rank 0's slab) against the reference
    ref_out, cb = None, None
    if rank == 0 and not args.no_cpu_baseline and world == 1:   # rank 0 at N = 1 only
        cb, ref_out = cpu_baseline_sample()
    elif rank == 0 and not args.no_parity:
        from oracle.oracle import Blocks, Reference   # the checker, after the timed region
        q = max(1, int(np.floor(np.sqrt(len(os.sched_getaffinity(0))))))
        A = Blocks(sz, sz, abi, abj, av)
        B = Blocks(sz, sz, bbi_all, bbj_all, bv_all)
        ref_out, _, _ = Reference().multiply(A, B, Blocks.empty(sz, sz), "cannon", q, q * q)
    parity = None
    if ref_out is not None:
        parity = parity_vs_reference(c if world == 1 else c.local(rank), ref_out)

    line = None
    if rank == 0:
        dist_desc = ("single GPU" if world == 1 else
                     f"case 2 weak scaling: A/C 400-block-row slabs per rank, B K-slabs "
                     f"gathered over NVLink/NCCL each step ({world} ranks)")
        line = {
            "metric": METRIC,
            "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": DATA,
            "config": bench_config(world, stats[-1]["products"], flops_step),
            "distribution": dist_desc,
            "roofline": {
                "bound": "tensor", "achieved": round(achieved, 3),
                "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(achieved / FP64_PEAK_TFLOPS, 4),
                "traffic": NCU_TRAFFIC_BYTES if world == 1 else None,
                "traffic_note": "DRAM bytes per launch (ncu); algorithmic bytes "
                                f"{alg_bytes / 1e9:.3f} GB (8*(|A|+|B|+|C|) unpadded elements "
                                "+ 12 B index per block)",
                "kernel": "k_smm_dmma<3,3,4,1> (FP64 DMMA 8x8x4 small-GEMM, T8 tiles, "
                          "bulk-async staged)",
                "peak_source": "measured FP64 DMMA/DFMA peak on B200 "
                               "(profiles/fp64_peak_r01.txt)",
                "step_share": round(kn_ms / ms_local, 3),
            },
            "e2e": {"value": round(e2e_val, 2), "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(kernels),
            "clocks": clocks.summary(),
        }
        if parity is not None:
            line["parity"] = parity
        if cb is not None:
            line["cpu_baseline"] = cb
    if world > 1:
        comm.close()
    else:
        for x in (a, b, c):
            x.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()
    if line is not None:   # last: after NCCL's teardown output
        print(json.dumps(line), flush=True)
        if parity is not None and not parity["ok"]:
            sys.exit("bench.py: parity check against the reference FAILED")


if __name__ == "__main__":
    main()
