"""dev: the reference's own algorithms on c1 with the host's threads (which one
is fastest on this box): Cannon on the largest square grid, case 1 / case 2 on
all cores."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from oracle.oracle import Blocks, Reference
ref = Reference()
cores = os.cpu_count()
sz = np.full(bench.NB, bench.BS, np.int32)
abi, abj, av = bench.make_blocks(bench.SEED_A, 400, 400, 23, 0.1)
bbi, bbj, bv = bench.make_blocks(bench.SEED_B, 400, 400, 23, 0.1)
A, B = Blocks(sz, sz, abi, abj, av), Blocks(sz, sz, bbi, bbj, bv)
flops = bench.useful_flops_host(abi, abj, bbi, bbj, 23)
q = int(np.floor(np.sqrt(cores)))
for algo, gq, P in (("cannon", q, q * q), ("case1", 1, cores), ("case2", 1, cores)):
    ts = []
    for _ in range(2):
        _, secs, _ = ref.multiply(A, B, Blocks.empty(sz, sz), algo, gq, P)
        ts.append(secs)
    print(f"{algo} P={P}: {min(ts)*1e3:.1f} ms = {flops/min(ts)/1e9:.1f} GFLOP/s", flush=True)
