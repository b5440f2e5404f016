"""dev: time the pieces of the e2e step (put A, put B, multiply, export)."""
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
cout = torch.empty(400 * 400 * 529, dtype=torch.float64).pin_memory()
for it in range(5):
    t = [time.perf_counter()]
    a = LocalStore(ctx, sz, sz); a.put_blocks(abi, abj, av_pin); ctx.sync(); t.append(time.perf_counter())
    b = LocalStore(ctx, sz, sz); b.put_blocks(bbi, bbj, bv_pin); ctx.sync(); t.append(time.perf_counter())
    c = LocalStore(ctx, sz, sz); multiply_local(ctx, a, b, c); ctx.sync(); t.append(time.perf_counter())
    ci, cj, _ = c.export(cout); ctx.sync(); t.append(time.perf_counter())
    for x in (a, b, c): x.close()
    t.append(time.perf_counter())
    d = np.diff(t) * 1e3
    print("putA %.2f putB %.2f mult %.2f export %.2f close %.2f  total %.2f ms" % (*d, sum(d)), flush=True)
