"""dev: raw host<->device copy bandwidth on this box (pinned and pageable)."""
import time, torch
n = 667 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
hp = torch.empty(n, dtype=torch.uint8)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, src, dst in (("h2d pinned", h, d), ("d2h pinned", d, h), ("h2d pageable", hp, d), ("d2h pageable", d, hp)):
    for _ in range(2):
        dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{name}: {n / dt / 1e9:.1f} GB/s ({dt*1e3:.2f} ms)", flush=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize(); t = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2 = h.copy_(d[:n], non_blocking=True) if False else None
torch.cuda.synchronize()
import os; print("cpus", os.cpu_count())
