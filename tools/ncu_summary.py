import csv, sys, subprocess
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]; v = r[2] if len(r) > 2 else r[1]
want = ['Kernel Name','gpu__time_duration.sum','dram__bytes_read.sum','dram__bytes_write.sum','gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
 'sm__warps_active.avg.per_cycle_active','launch__registers_per_thread','launch__occupancy_limit_registers','launch__occupancy_limit_shared_mem',
 'sm__throughput.avg.pct_of_peak_sustained_elapsed','lts__t_sector_hit_rate.pct','smsp__issue_active.avg.pct_of_peak_sustained_active',
 'sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active','lts__throughput.avg.pct_of_peak_sustained_elapsed',
 'l1tex__throughput.avg.pct_of_peak_sustained_active','launch__grid_size','launch__block_size']
for k in want:
    if k in h: print(f"{k:75s} {v[h.index(k)]}")
rows = []
for i, k in enumerate(h):
    if 'pcsamp_warps_issue_stalled' in k and not k.endswith('not_issued'):
        try: rows.append((float(v[i]), k))
        except: pass
tot = sum(x for x, _ in rows) or 1
print("top stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')} {100*x/tot:.0f}%" for x, k in sorted(rows, reverse=True)[:6]))
