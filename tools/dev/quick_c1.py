"""Quick timing of the local multiply on a c1-like shape (dev tool):
  python tools/quick_c1.py [block_size] [n_blocks] [occupancy]
Inputs: bench.make_blocks (numpy PCG64, seeds 1001/1002)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_1910_13555_b200.store import Context, LocalStore, multiply_local

bs = int(sys.argv[1]) if len(sys.argv) > 1 else 23
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 400
occ = float(sys.argv[3]) if len(sys.argv) > 3 else 0.10
sz = np.full(nb, bs, np.int32)
t = time.time()
abi, abj, av = bench.make_blocks(bench.SEED_A, nb, nb, bs, occ)
bbi, bbj, bv = bench.make_blocks(bench.SEED_B, nb, nb, bs, occ)
print("gen", time.time() - t, len(abi), len(bbi), flush=True)
ctx = Context(0)
ctx.set_timing(True)
a = LocalStore(ctx, sz, sz); a.put_blocks(abi, abj, av)
b = LocalStore(ctx, sz, sz); b.put_blocks(bbi, bbj, bv)
c = LocalStore(ctx, sz, sz)
for it in range(8):
    c.clear(); ctx.sync()
    t0 = time.perf_counter()
    st = multiply_local(ctx, a, b, c)
    ctx.sync()
    dt = time.perf_counter() - t0
    print(f"iter {it}: {dt*1e3:.3f} ms  {st['flops']/dt/1e9:.1f} GFLOP/s  numeric {st['ms_numeric']:.3f} ms = {st['flops']/st['ms_numeric']/1e9:.1f} GFLOP/s total-dev {st['ms_total']:.3f} ms  products {st['products']} kernels {st['kernels']}", flush=True)
