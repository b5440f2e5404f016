"""dev: put_blocks breakdown."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1910_13555_b200.store import Context, LocalStore, multiply_local
ctx = Context(0)
sz = np.full(bench.NB, bench.BS, np.int32)
abi, abj, av = bench.make_blocks(bench.SEED_A, 400, 400, 23, 0.1)
av_pin = torch.from_numpy(av).pin_memory()
T = lambda: (ctx.sync(), time.perf_counter())[1]
for it in range(6):
    t0 = T(); a = LocalStore(ctx, sz, sz); t1 = T()
    a.put_blocks(abi, abj, av_pin); t2 = T()
    a.clear(); t3 = T()
    a.put_blocks(abi, abj, av); t4 = T()   # pageable numpy source
    a.close(); t5 = T()
    print("create %.2f put(pinned) %.2f clear %.2f put(pageable) %.2f close %.2f ms" %
          tuple(1e3 * x for x in (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)), flush=True)
