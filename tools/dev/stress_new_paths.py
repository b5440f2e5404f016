"""Ad-hoc stress of the round-2 paths (WIDE, warp-row fill, split-count, 128-thread pass 1):
N random cases against the oracle.  python tools/dev/stress_new_paths.py [N]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    from oracle.oracle import Oracle
    from helpers import assert_parity, from_store, to_store
    from paper_1910_13555_b200.store import Context, multiply_local
    oracle = Oracle()
    ctx = Context(0)
    variants = [("BT_WARP_ROWS", "128"), ("BT_WARP_ROWS", "256"), ("BT_FILL_SPLITS", "3"),
                ("BT_COUNT_THREADS", "128"), ("BT_WIDE", "1")]
    for seed in range(n):
        rng = np.random.default_rng(50000 + seed)
        k, v = variants[seed % len(variants)]
        os.environ[k] = v
        pal = lambda hi: rng.choice(np.arange(1, hi + 1), size=int(rng.integers(1, 4)), replace=False)  # noqa
        pm, pk, pn = pal(100), pal(100), pal(100)
        if seed % 3 == 0:
            pm = np.append(pm, rng.choice([169, 299]))
        rsz = rng.choice(pm, int(rng.integers(2, 50))).astype(np.int32)
        ksz = rng.choice(pk, int(rng.integers(2, 200))).astype(np.int32)
        nsz = rng.choice(pn, int(rng.integers(2, 50))).astype(np.int32)
        scale = float(rng.choice([0.0, 6.0]))
        A = oracle.random_matrix(60000 + seed, rsz, ksz, float(rng.choice([0.02, 0.1, 0.4, 0.8])), scale)
        B = oracle.random_matrix(70000 + seed, ksz, nsz, float(rng.choice([0.02, 0.1, 0.4])), scale)
        Cin = oracle.random_matrix(80000 + seed, rsz, nsz, float(rng.choice([0.0, 0.3])), scale)
        eps = 1e-3 if scale else 0.0
        want, nprod, flops = oracle.multiply(A, B, Cin, eps)
        a, b, c = to_store(ctx, A), to_store(ctx, B), to_store(ctx, Cin)
        st = multiply_local(ctx, a, b, c, eps)
        assert st["products"] == nprod and st["flops"] == flops, (seed, k, v)
        assert_parity(from_store(c), want)
        for s in (a, b, c):
            s.close()
        del os.environ[k]
    ctx.close()
    print(f"stress: {n} cases ok", flush=True)


if __name__ == "__main__":
    main()
