"""Quick timing of the local multiply on BASELINE config 1 (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle.oracle import Oracle
from paper_1910_13555_b200.store import Context, LocalStore, multiply_local

o = Oracle()
bs = int(sys.argv[1]) if len(sys.argv) > 1 else 23
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 400
occ = float(sys.argv[3]) if len(sys.argv) > 3 else 0.10
sz = np.full(nb, bs, np.int32)
t = time.time()
A = o.random_matrix(1001, sz, sz, occ)
B = o.random_matrix(1002, sz, sz, occ)
print("gen", time.time() - t, A.nblk, B.nblk, flush=True)
ctx = Context(0)
ctx.set_timing(True)
a = LocalStore(ctx, sz, sz); a.put_blocks(A.bi, A.bj, A.vals)
b = LocalStore(ctx, sz, sz); b.put_blocks(B.bi, B.bj, B.vals)
c = LocalStore(ctx, sz, sz)
for it in range(8):
    c.clear(); ctx.sync()
    t0 = time.perf_counter()
    st = multiply_local(ctx, a, b, c)
    ctx.sync()
    dt = time.perf_counter() - t0
    print(f"iter {it}: {dt*1e3:.3f} ms  {st['flops']/dt/1e9:.1f} GFLOP/s  numeric {st['ms_numeric']:.3f} ms = {st['flops']/st['ms_numeric']/1e9:.1f} GFLOP/s total-dev {st['ms_total']:.3f} ms  products {st['products']} kernels {st['kernels']}", flush=True)
