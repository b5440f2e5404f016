"""dev: all-gather of per-GPU slabs by copy-engine peer copies (one process, all
visible GPUs): each GPU pulls every peer's slab on its own stream."""
import sys, time, torch
n = torch.cuda.device_count()
mb = float(sys.argv[1]) if len(sys.argv) > 1 else 18.4
nel = int(mb * 1e6 / 8)
src = [torch.randn(nel, dtype=torch.float64, device=f"cuda:{d}") for d in range(n)]
dst = [torch.empty(n * nel, dtype=torch.float64, device=f"cuda:{d}") for d in range(n)]
streams = {(d, p): torch.cuda.Stream(device=d) for d in range(n) for p in range(n)}
def run():
    for d in range(n):
        for p in range(n):
            with torch.cuda.stream(streams[(d, p)]):
                dst[d][p * nel:(p + 1) * nel].copy_(src[p], non_blocking=True)
    for d in range(n):
        torch.cuda.synchronize(d)
for _ in range(3): run()
t = time.perf_counter()
for _ in range(10): run()
dt = (time.perf_counter() - t) / 10
print(f"{n} GPUs, {mb} MB per slab: {dt*1e6:.1f} us per all-gather, "
      f"{(n-1)*nel*8/dt/1e9:.1f} GB/s received per GPU")
