"""Summarise an ncu --set full report: key metrics + stall samples by source line."""
import csv, collections, re, subprocess, sys
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'launch__registers_per_thread', 'launch__occupancy_limit_registers', 'launch__occupancy_limit_shared_mem',
        'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__cycles_elapsed.avg', 'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'smsp__issue_active.avg.pct_of_peak_sustained_active']
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:62s} {units[i]:8s}", [d[i][:40] for d in data])
stalls = [h for h in hdr if h.startswith('smsp__average_warps_issue_stalled') and h.endswith('per_issue_active.ratio')]
vals = {h: [float(d[hdr.index(h)] or 0) for d in data] for h in stalls}
print("stalls (per issue):", ", ".join(f"{h.split('stalled_')[1].split('_per')[0]}={v[0]:.2f}/{v[-1]:.2f}"
                                      for h, v in sorted(vals.items(), key=lambda x: -x[1][0]) if v[0] > 0.05))
