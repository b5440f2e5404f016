"""Regenerates the golden fixtures from the compiled reference (oracle/_ref).

Run where /root/reference exists (make -C oracle ref first):
    python tests/golden/make_golden.py
Each fixture is the reference's multiply_dispatch output on seeded inputs
(random_matrix, oracles.hpp:74-85), plus the per-rank ledger, stored as .npz.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import Oracle, Reference  # noqa: E402

CASES = [
    # name, seed, row sizes, inner sizes, col sizes, occ A, occ B, occ C, algo, q, nprocs
    ("c1_small", 11, [23] * 24, [23] * 24, [23] * 24, 0.10, 0.10, 0.0, "cannon", 1, 1),
    ("mixed_cannon2", 12, [3, 5, 2, 7, 1, 4, 6, 2], [2, 6, 3, 5, 4, 1], [4, 1, 3, 6, 2], 0.5,
     0.5, 0.2, "cannon", 2, 4),
    ("mixed_cannon3", 13, [5, 13, 23, 5, 13, 23, 5, 13, 23], [13, 5, 23, 13, 5, 23],
     [23, 13, 5, 23, 13, 5, 23], 0.4, 0.4, 0.1, "cannon", 3, 9),
    ("tall_case1", 14, [20] * 4, [20] * 64, [20] * 4, 0.3, 0.3, 0.2, "case1", 1, 4),
    ("tall_case2", 15, [20] * 64, [20] * 4, [20] * 4, 0.3, 0.3, 0.2, "case2", 1, 4),
    ("dense_cannon2", 16, [4] * 8, [4] * 8, [4] * 8, 1.0, 1.0, 0.0, "cannon", 2, 4),
]


def main():
    o, r = Oracle(), Reference()
    index = {}
    for name, seed, rs, ks, ns, oa, ob, oc, algo, q, p in CASES:
        A = o.random_matrix(seed, rs, ks, oa)
        B = o.random_matrix(seed + 1000, ks, ns, ob)
        Cin = o.random_matrix(seed + 2000, rs, ns, oc)
        out, _, ledger = r.multiply(A, B, Cin, algo, q, p)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"),
                            rsz=np.asarray(rs, np.int32), ksz=np.asarray(ks, np.int32),
                            nsz=np.asarray(ns, np.int32), c_bi=out.bi, c_bj=out.bj,
                            c_vals=out.vals)
        index[name] = dict(seed=seed, occ=[oa, ob, oc], algo=algo, grid_q=q, nprocs=p,
                           seeds=[seed, seed + 1000, seed + 2000], nblk=int(out.nblk),
                           ledger={str(k): v for k, v in ledger.items()})
    with open(os.path.join(HERE, "index.json"), "w") as f:
        json.dump(index, f, indent=1, sort_keys=True)
    print("wrote", len(index), "fixtures")


if __name__ == "__main__":
    main()
