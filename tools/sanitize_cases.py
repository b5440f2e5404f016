"""Small invocations of every numeric/symbolic kernel path, for
compute-sanitizer (racecheck / memcheck / synccheck / initcheck, one tool per
run):

  compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Paths: k_smm_dmma single class, MULTI (mixed sizes, one launch), WIDE (blocks
wider than 32 / k > 64), the warp-row fill, PANELS (K
panels in one launch: cross-CTA acquire/release flags), generic (n > 32),
the eps filter + norms, column-chunked symbolic passes, split fill CTAs, the
asynchronous export, the tensor remap.  Inputs: numpy, seeded; no checking
here (parity lives in tests/)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1910_13555_b200.store import Context, LocalStore, multiply_local  # noqa: E402


def rand(rng, rsz, csz, occ):
    mask = rng.random((len(rsz), len(csz))) < occ
    bi, bj = np.nonzero(mask)
    vals = rng.standard_normal(int(np.sum(rsz[bi].astype(np.int64) * csz[bj])))
    return bi.astype(np.int64), bj.astype(np.int64), vals


def run(ctx, rng, rsz, ksz, nsz, occ=0.3, eps=0.0, env=None):
    old = {}
    for k, v in (env or {}).items():
        old[k] = os.environ.get(k)
        os.environ[k] = v
    a, b, c = LocalStore(ctx, rsz, ksz), LocalStore(ctx, ksz, nsz), LocalStore(ctx, rsz, nsz)
    a.put_blocks(*rand(rng, rsz, ksz, occ))
    b.put_blocks(*rand(rng, ksz, nsz, occ))
    c.put_blocks(*rand(rng, rsz, nsz, 0.1))
    st = multiply_local(ctx, a, b, c, eps)
    c.export()
    for k, v in old.items():
        if v is None:
            os.environ.pop(k)
        else:
            os.environ[k] = v
    print(f"{env or {}}: {st['products']} products, {st['kernels']} kernels", flush=True)
    return c


def main():
    ctx = Context(0)
    rng = np.random.default_rng(1)
    u = lambda n, s: np.full(n, s, np.int32)  # noqa: E731
    mix = lambda n: np.array([5, 13, 23], np.int32)[rng.integers(0, 3, n)]  # noqa: E731
    run(ctx, rng, u(12, 23), u(12, 23), u(12, 23))                          # one class
    run(ctx, rng, mix(20), mix(20), mix(20), eps=1.0)                       # MULTI + eps
    run(ctx, rng, u(10, 20), u(60, 20), u(10, 20), occ=0.3,
        env={"BT_KPANELS": "3"})                                             # PANELS fused
    run(ctx, rng, mix(10), mix(60), mix(10), env={"BT_KPANELS": "3"})       # panels per launch
    run(ctx, rng, np.array([37, 40, 5], np.int32), np.array([13, 40], np.int32),
        np.array([37, 8], np.int32), occ=0.8, env={"BT_WIDE": "0"})          # generic
    run(ctx, rng, np.array([37, 100, 5], np.int32), np.array([13, 70, 130], np.int32),
        np.array([41, 8, 64], np.int32), occ=0.8)                            # WIDE (tiles, k slices)
    run(ctx, rng, u(8, 48), u(40, 40), u(8, 48), occ=0.5,
        env={"BT_KPANELS": "3"})                                             # WIDE per panel
    run(ctx, rng, mix(40), mix(40), mix(40), occ=0.02, env={"BT_WARP_ROWS": "256"})  # warp-row fill
    run(ctx, rng, mix(8), mix(300), mix(200), occ=0.1, env={"BT_COLW": "40"})   # column chunks
    run(ctx, rng, mix(6), mix(2000), mix(30), occ=0.2, env={"BT_FILL_SPLITS": "3"})  # split fill
    c = run(ctx, rng, mix(30), mix(30), mix(30))
    nb, ne = c.info()
    buf = np.zeros(ne)
    c.export(buf, asynchronous=True)
    ctx.sync()
    c.filter(0.5)
    c.norms()
    from paper_1910_13555_b200.tensor import SparseTensor
    s = [np.array([2, 3], np.int32), np.array([4, 1, 2], np.int32), np.array([3, 3], np.int32)]
    t = SparseTensor(ctx, s, [0, 1], [2])
    t.store.put_blocks(*rand(rng, np.asarray(t.store.rsz), np.asarray(t.store.csz), 0.5))
    t.remap([2], [1, 0])
    ctx.close()
    print("sanitize cases done", flush=True)


if __name__ == "__main__":
    main()
