"""dev: do H2D and D2H copies on two streams overlap on this box?  Times a
667 MB D2H alone, a 68 MB H2D alone, and both issued together (pinned)."""
import time, torch
nd, nu = 667 << 20, 68 << 20
hd = torch.empty(nd, dtype=torch.uint8).pin_memory()
dd = torch.empty(nd, dtype=torch.uint8, device="cuda")
hu = torch.empty(nu, dtype=torch.uint8).pin_memory()
du = torch.empty(nu, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(which):
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t = time.perf_counter()
    if "d2h" in which:
        with torch.cuda.stream(s1):
            e[0].record(); hd.copy_(dd, non_blocking=True); e[1].record()
    if "h2d" in which:
        with torch.cuda.stream(s2):
            e[2].record(); du.copy_(hu, non_blocking=True); e[3].record()
    torch.cuda.synchronize()
    out = {"wall_ms": round((time.perf_counter() - t) * 1e3, 2)}
    if "d2h" in which: out["d2h_ms"] = round(e[0].elapsed_time(e[1]), 2)
    if "h2d" in which: out["h2d_ms"] = round(e[2].elapsed_time(e[3]), 2)
    return out
for w in ("d2h", "h2d", "d2h+h2d", "d2h+h2d"):
    print(w, run(w), flush=True)
