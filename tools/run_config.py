"""Run one BASELINE.json config on the GPU and time the block-sparse multiply.

  python tools/run_config.py c2|c3|c4 [--steps K] [--occ X]

Inputs are synthetic and seeded (numpy PCG64).  Full-size parity of the same
inputs against the oracle lives in tests/test_configs_gpu.py (the oracle is
test infrastructure and is not imported here).  c1 is bench.py's workload; c5
has its own driver (tools/run_c5.py).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def blocks_random(rng, rsz, csz, occ, scale_exp=0.0, band=None):
    """(bi, bj, vals) canonical; presence Bernoulli(occ) (or |i-j| <= band), N(0,1)
    values, optionally scaled per block by 10^(-scale_exp*u)."""
    nbr, nbc = len(rsz), len(csz)
    if band is not None:
        mask = np.abs(np.arange(nbr)[:, None] - np.arange(nbc)[None, :]) <= band
    else:
        mask = rng.random((nbr, nbc)) < occ
    bi, bj = np.nonzero(mask)
    sizes = rsz[bi].astype(np.int64) * csz[bj]
    vals = rng.standard_normal(int(sizes.sum()))
    if scale_exp > 0:
        scale = 10.0 ** (-scale_exp * rng.random(len(bi)))
        vals *= np.repeat(scale, sizes)
    return bi.astype(np.int64), bj.astype(np.int64), vals


def config(name, rng, occ=None):
    """returns (rsz, ksz, nsz, A, B, eps, description)"""
    if name == "c1":
        sz = np.full(400, 23, np.int32)
        A = blocks_random(rng, sz, sz, 0.10)
        B = blocks_random(rng, sz, sz, 0.10)
        return sz, sz, sz, A, B, 0.0, "c1: 400x400 blocks of 23x23, occ 0.10 (bench.py's workload shape)"
    if name == "c2":
        sizes = np.array([5, 13, 23], np.int32)[rng.integers(0, 3, 1463)]
        A = blocks_random(rng, sizes, sizes, 0.01, 12.0)
        B = blocks_random(rng, sizes, sizes, 0.01, 12.0)
        return sizes, sizes, sizes, A, B, 1e-8, (
            f"c2: mixed {{5,13,23}} basis, {len(sizes)} blocks (N={int(sizes.sum())}), "
            "occ 0.01, per-block scale 10^(-12u), eps 1e-8")
    if name == "c3":
        m = np.full(100, 20, np.int32)
        k = np.full(20000, 20, np.int32)
        o = 0.10 if occ is None else occ
        A = blocks_random(rng, m, k, o)
        B = blocks_random(rng, k, m, o)
        return m, k, m, A, B, 0.0, ("c3: C 2000x2000 = A 2000x400000 * B 400000x2000, "
                                    f"blocks 20, occ {o:.2f} (single GPU, local multiply)")
    if name == "c4":
        ao = np.tile(np.array([13, 23], np.int32), 100)       # a, b: 200 AO blocks
        aux = np.tile(np.array([13, 23], np.int32), 200)      # P, Q: 400 aux blocks
        rows = np.multiply.outer(ao, ao).ravel().astype(np.int32)  # (ab) matricized, b fastest
        T = blocks_random(rng, rows, aux, 0.001)
        M = blocks_random(rng, aux, aux, 0.0, band=7)
        return rows, aux, aux, T, M, 0.0, ("c4: (ab|P)(P|Q), a,b 200 AO blocks, P,Q 400 aux "
                                           "blocks, 13/23 alternating, T occ 0.001, (P|Q) band 7")
    if name in ("big64", "big40"):
        # not a BASELINE config: blocks wider than the DMMA tile kernels take
        # (n > 32): the generic kernel's workload
        bs = int(name[3:])
        sz = np.full(200, bs, np.int32)
        o = 0.1 if occ is None else occ
        A = blocks_random(rng, sz, sz, o)
        B = blocks_random(rng, sz, sz, o)
        return sz, sz, sz, A, B, 0.0, f"{name}: 200x200 blocks of {bs}x{bs}, occ {o}"
    if name in ("tiny5", "tiny3", "tiny1"):
        # not a BASELINE config: uniform tiny blocks, ~20 products per C block
        # (compute-heavy), the DFMA-vs-DMMA A/B workload (BT_DFMA=0/1)
        bs = int(name[4:])
        nb = {5: 2000, 3: 2400, 1: 4000}[bs]
        o = {5: 0.01, 3: 0.01, 1: 0.005}[bs] if occ is None else occ
        sz = np.full(nb, bs, np.int32)
        A = blocks_random(rng, sz, sz, o)
        B = blocks_random(rng, sz, sz, o)
        return sz, sz, sz, A, B, 0.0, (f"{name}: {nb}x{nb} blocks of {bs}x{bs}, occ {o}")
    raise SystemExit(f"unknown config {name}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--no-check", action="store_true", help="(accepted; parity is in tests/)")
    ap.add_argument("--occ", type=float, default=None, help="c3: block occupancy (0.10-0.50)")
    args = ap.parse_args()
    import torch
    from paper_1910_13555_b200.store import Context, LocalStore, multiply_local
    rng = np.random.default_rng(2024)
    t0 = time.time()
    rsz, ksz, nsz, A, B, eps, desc = config(args.config, rng, args.occ)
    gen_s = time.time() - t0
    ctx = Context(0)
    # events around the kernels, no wait inside the call (as bench.py): the
    # step time ends with the last kernel, not with the host's return
    ctx.set_timing(2 if os.environ.get("BT_PHASES") is None else 1)
    a = LocalStore(ctx, rsz, ksz)
    a.put_blocks(*A)
    b = LocalStore(ctx, ksz, nsz)
    b.put_blocks(*B)
    c = LocalStore(ctx, rsz, nsz)
    stream = torch.cuda.ExternalStream(ctx.stream)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    times, nums, st = [], [], None
    for it in range(2 + args.steps):
        c.clear()
        with torch.cuda.stream(stream):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        st = multiply_local(ctx, a, b, c, eps)
        with torch.cuda.stream(stream):
            e1.record(stream)
        num = ctx.last_timing()[0]
        torch.cuda.synchronize()
        if it >= 2:
            times.append(e0.elapsed_time(e1))
            nums.append(num)
    ms = float(np.median(times))
    st["ms_numeric"] = float(np.median(nums))
    a_el = int(a.info()[1]); b_el = int(b.info()[1]); c_el = int(c.info()[1])
    bytes_alg = 8 * (a_el + b_el + c_el)
    out = {"config": args.config, "workload": desc, "products": st["products"],
           "candidates": st["candidates"], "useful_gflop": st["flops"] / 1e9,
           "c_blocks": st["c_blocks_out"], "ms_median": round(ms, 4),
           "gflops": round(st["flops"] / ms / 1e6, 1),
           "numeric_ms": round(st["ms_numeric"], 4),
           "numeric_tflops": round(st["flops"] / st["ms_numeric"] / 1e9, 3),
           "alg_bytes": bytes_alg, "alg_gbs": round(bytes_alg / ms / 1e6, 1),
           "ai_flop_per_byte": round(st["flops"] / bytes_alg, 2), "gen_s": round(gen_s, 1)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
