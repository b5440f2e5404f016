"""dev: host-side time of each call of the pipelined e2e step (async export),
no syncs inside the loop except the library's own."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1910_13555_b200.store import Context, LocalStore, multiply_local
ctx = Context(0)
sz = np.full(bench.NB, bench.BS, np.int32)
abi, abj, av = bench.make_blocks(bench.SEED_A, 400, 400, 23, 0.1)
bbi, bbj, bv = bench.make_blocks(bench.SEED_B, 400, 400, 23, 0.1)
av_pin = torch.from_numpy(av).pin_memory(); bv_pin = torch.from_numpy(bv).pin_memory()
couts = [torch.empty(400 * 400 * 529, dtype=torch.float64).pin_memory() for _ in range(2)]
a, b, c = (LocalStore(ctx, sz, sz) for _ in range(3))
t00 = time.perf_counter()
for it in range(8):
    t = [time.perf_counter()]
    a.clear(); b.clear(); c.clear(); t.append(time.perf_counter())
    a.put_blocks(abi, abj, av_pin); t.append(time.perf_counter())
    b.put_blocks(bbi, bbj, bv_pin); t.append(time.perf_counter())
    multiply_local(ctx, a, b, c); t.append(time.perf_counter())
    ci, cj, _ = c.export(couts[it % 2], asynchronous=True); t.append(time.perf_counter())
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("clear %.2f putA %.2f putB %.2f mult %.2f export %.2f - %.2f  total %.2f ms" % (*d, sum(d)), flush=True)
ctx.sync()
print("all %.2f ms/step" % ((time.perf_counter() - t00) * 1e3 / 8))
