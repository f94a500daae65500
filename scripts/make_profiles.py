"""Summarise gpurun_out ncu captures into profiles/ (tracked)."""
import csv, collections, json, subprocess, sys, os
tag = sys.argv[1]
out_dir = "profiles"
def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    return rows[0], rows[1], rows[2:]
lines = [f"# ncu summary, {tag}\n"]
summary = {}
GRID = {"c2": 2048, "wet": 2048, "c5": 8192}
for cfg in ("c2", "wet", "c5"):
    rep = f"gpurun_out/prof_{tag}_{cfg}.ncu-rep"
    if not os.path.exists(rep):
        continue
    n = GRID[cfg]
    # processed-tile fraction of the captured run (bench.py's JSON line in the ncu log)
    frac = None
    try:
        for ln in open(f"gpurun_out/prof_{tag}_{cfg}.log"):
            if ln.startswith("{"):
                frac = json.loads(ln)["roofline"]["processed_tile_frac"]
    except Exception:
        pass
    hdr, units, data = raw(rep)
    g = lambda r, k: r[hdr.index(k)] if k in hdr else ""
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
            "launch__grid_size", "launch__block_size"]
    lines.append(f"\n## {cfg} {n}x{n} (bench.py --config {'c2' if cfg == 'c5' else cfg} --ncols {n} --nrows {n}), "
                 f"`ncu --set full --clock-control none`\n")
    lines.append("| metric | unit | " + " | ".join(g(r, "Kernel Name")[:40] for r in data) + " |")
    lines.append("|---|---|" + "---|" * len(data))
    for k in keys:
        if k in hdr:
            lines.append(f"| {k} | {units[hdr.index(k)]} | " + " | ".join(g(r, k) for r in data) + " |")
    stalls = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
    top = sorted(stalls, key=lambda h: -float(data[0][hdr.index(h)] or 0))[:8]
    lines.append("\nTop stall reasons (warps stalled per issue, pred/corr): " +
                 ", ".join(f"{h.split('stalled_')[1].split('_per')[0]} {float(data[0][hdr.index(h)]):.2f}/{float(data[-1][hdr.index(h)]):.2f}" for h in top))
    def tobytes(r, k):
        v = float(g(r, k)); u = units[hdr.index(k)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    traffic = sum(tobytes(r, "dram__bytes_read.sum") + tobytes(r, "dram__bytes_write.sum") for r in data)
    pct = lambda k: [round(float(g(r, k)), 2) for r in data] if k in hdr else None  # noqa: E731
    alg = 464 * n * n
    alg_proc = (208 * frac[0] + 256 * frac[1]) * n * n if frac else None
    summary[cfg] = {"config": "c2" if cfg == "c5" else cfg, "grid": [n, n], "dram_bytes_per_step": traffic,
                    "alg_bytes_per_step": alg, "processed_tile_frac": frac,
                    "alg_bytes_processed_tiles_per_step": alg_proc,
                    "kernels": [g(r, "Kernel Name") for r in data],
                    "fp64_pipe_active_pct": pct("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                    "issue_active_pct": pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                    "dram_throughput_pct": pct("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
    lines.append(f"\nDRAM traffic per step (pred+corr): {traffic/1e6:.1f} MB; algorithmic 464 B x {n}^2 = "
                 f"{alg/1e6:.1f} MB (ratio {traffic/alg:.3f})" +
                 (f"; algorithmic bytes of the processed tiles ({frac[0]:.3f}/{frac[1]:.3f} of the tiles) = "
                  f"{alg_proc/1e6:.1f} MB (ratio {traffic/alg_proc:.3f})" if alg_proc else "") + ".\n")
# launch list
lc = f"gpurun_out/launches_{tag}.csv"
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        agg[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    lines.append("\n## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, "
                 "bench.py --steps 8 --warmup 3, cold-cache serialised: compare shares)\n")
    lines.append("| kernel | launches | mean us | share |")
    lines.append("|---|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| {k} | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {100*sum(v)/tot:.1f}% |")
# instruction ceilings from the fully wet capture (every tile processed: per cell-update counts
# are exact): FP64-pipe thread instructions (DADD, DMUL, DFMA, DSETP) and all thread
# instructions of both stage kernels, from the SASS source page
iroof = None
rep = f"gpurun_out/prof_{tag}_wet.ncu-rep"
if os.path.exists(rep):
    import re
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout.split("\n")
    blocks, cur = [], None
    for ln in txt:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]; blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    fp64 = allt = 0
    seen = set()
    for b in blocks:
        if b[0] in seen:
            continue
        seen.add(b[0])
        rows = list(csv.reader(b[1:])); hdr = rows[0]
        ti = hdr.index("Thread Instructions Executed")
        for r in rows[1:]:
            if len(r) != len(hdr):
                continue
            op = re.sub(r'^@!?U?P\w+\s+', '', r[1].strip()).split(' ')[0].split('.')[0]
            allt += int(r[ti])
            if op in ("DADD", "DMUL", "DFMA", "DSETP"):
                fp64 += int(r[ti])
    cells = GRID["wet"] ** 2
    peaks = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    f_cu, t_cu = fp64 / cells, allt / cells
    iroof = {"fp64_thread_ops_per_cell_update": round(f_cu, 1), "thread_instructions_per_cell_update": round(t_cu, 1),
             "fp64_ceiling_gcups": round(148 * 64 * clk / f_cu / 1e9, 3),
             "issue_ceiling_gcups": round(148 * 128 * clk / t_cu / 1e9, 3),
             "how": "fully wet 2048^2 capture, both stage kernels; 64 FP64 and 128 thread instructions "
                    "per clock per SM, 148 SMs, sm_max_mhz"}
    lines.append(f"\n## Instruction ceilings (fully wet capture)\n\n{json.dumps(iroof)}\n")
if "c2" in summary:
    d = summary["c2"]; d["wet"] = summary.get("wet"); d["c5"] = summary.get("c5"); d["source"] = f"profiles/{tag}_ncu.md"
    d["instruction_roofline"] = iroof
    json.dump(d, open(f"{out_dir}/ncu_stage_summary.json", "w"), indent=1)
open(f"{out_dir}/{tag}_ncu.md", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
