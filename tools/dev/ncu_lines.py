"""Per-source-line instruction and stall-sample shares of one kernel in an ncu report.
usage: ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, subprocess, sys, re, collections
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", "regex:" + kre, "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
cur, out, hd = None, [], None
for r in rows:
    if r and r[0] == "File Path": cur = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No": hd = r; continue
    if not r or r[0] in ("", "Function Name"): continue
    try:
        ln = int(r[0]); ex = float(r[7]) if r[7] not in ("-", "") else 0
        s = float(r[4]) if r[4] not in ("-", "") else 0
    except Exception:
        continue
    out.append((cur, ln, r[1][:100], ex, s))
te = sum(o[3] for o in out) or 1; ts = sum(o[4] for o in out) or 1
print(f"warp instructions {te:.0f}, stall samples {ts:.0f}")
for o in sorted(out, key=lambda o: -o[4])[:n]:
    print(f"{o[0][:14]:14s}{o[1]:5d} ex {o[3]/te*100:5.1f}% smp {o[4]/ts*100:5.1f}%  {o[2]}")
