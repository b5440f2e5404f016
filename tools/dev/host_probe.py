"""dev: host-side cost of the bench step's API calls (clear, multiply) on c1."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_1910_13555_b200.store import Context, LocalStore, multiply_local
ctx = Context(0)
ctx.set_timing(True)
sz = np.full(bench.NB, bench.BS, np.int32)
abi, abj, av = bench.make_blocks(bench.SEED_A, 400, 400, 23, 0.1)
bbi, bbj, bv = bench.make_blocks(bench.SEED_B, 400, 400, 23, 0.1)
a = LocalStore(ctx, sz, sz); a.put_blocks(abi, abj, av)
b = LocalStore(ctx, sz, sz); b.put_blocks(bbi, bbj, bv)
c = LocalStore(ctx, sz, sz)
stream = torch.cuda.ExternalStream(ctx.stream)
for it in range(12):
    ctx.sync()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    t1 = time.perf_counter()
    c.clear()
    t2 = time.perf_counter()
    st = multiply_local(ctx, a, b, c)
    t3 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"record {1e6*(t1-t0):.1f} us | clear {1e6*(t2-t1):.1f} us | multiply call {1e6*(t3-t2):.1f} us"
          f" (dev total {1e3*st['ms_total']:.1f}) | step events {1e3*e0.elapsed_time(e1):.1f} us", flush=True)
