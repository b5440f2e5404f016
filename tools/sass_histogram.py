"""Opcode histogram of the numeric / symbolic kernels in libbtcuda.so
(cuobjdump -sass): proves the FP64 tensor path (DMMA.8x8x4), the bulk-async
copy engine (UBLKCP + SYNCS mbarrier ops) and the cp.async staging (LDGSTS).
    python tools/sass_histogram.py [lib] > profiles/r02/sass_histogram.txt"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1910_13555_b200/libbtcuda.so"
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
KEEP = ("DMMA", "DFMA", "UBLKCP", "SYNCS", "LDGSTS", "LDS", "LDG", "STG", "STS", "BAR", "SHFL",
        "ATOM", "RED", "UTC")
total = collections.Counter()
rows = []
for f in re.split(r"\n\s*Function : ", txt)[1:]:
    name = f.split("\n", 1)[0].strip()
    ops = re.findall(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", f)
    c = collections.Counter(o if o.startswith(("DMMA", "UBLKCP", "SYNCS", "LDGSTS")) else
                            o.split(".")[0] for o in ops)
    for k, v in c.items():
        if k.startswith(("DMMA", "DFMA", "UBLKCP", "SYNCS", "LDGSTS", "UTC")):
            total[k] += v
    if "k_smm" in name or "k_row" in name or "k_remap_vals" in name:
        keys = sorted(k for k in c if k.startswith(KEEP))
        rows.append((name, len(ops), ", ".join(f"{k} {c[k]}" for k in keys)))
print(f"# SASS opcode histogram of {lib} (cuobjdump -sass, sm_100a)")
print("# no UTC*MMA: sm_100a has no FP64 tcgen05 kind; FP64 tensor math is DMMA.8x8x4")
for name, n, keys in rows:
    print(f"{name}\n    {n} instructions: {keys}")
print("\nwhole library:", ", ".join(f"{k} {v}" for k, v in sorted(total.items())))
