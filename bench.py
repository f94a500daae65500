#!/usr/bin/env python
"""bench.py — cell-updates/s (GCUPS) of the B200 time-stepping core.

Workload (BASELINE.json configs[1]): Mode-I release on the synthetic 2048x2048
valley DEM, FP64, one full accepted time step per "step" (apply_boundaries +
CFL reduction + Heun predictor + corrector, solver.cpp:637-649), inputs
resident in HBM, device-resident loop (tp_steps).  Unit of work: one interior
cell advanced one step; value = ncols*nrows*K / (max-over-ranks device time).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--config c2|wet|c1|c3|c4]

N>1 (launched by torchrun): weak scaling, each rank owns a 2048-row slab of a
2048 x (2048 N) valley (row-block decomposition, NCCL halo exchange, lambda
all-reduce — paper_2104_06784_b200/distributed.py).

The JSON line also carries: the stage kernels' roofline (algorithmic 464 B per
cell-update, against MEASURED_PEAKS.json hbm_gbs), the CPU
reference timed on this host (cpu_baseline), the end-to-end C-ABI number with
host<->device copies (e2e), clocks sampled during the timed region, and the
number of our kernels launched inside it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "cell-updates/sec (GCUPS) and % HBM roofline at 1/2/4/8 B200 vs host-CPU ref"
ALG_BYTES_PER_CELL_UPDATE = 464  # predictor 208 B + corrector 256 B (FP64)
ALG_BYTES_PRED = 208
ALG_BYTES_CORR = 256


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def scenario_for(name, ncols, nrows):
    from paper_2104_06784_b200 import scenarios
    if name == "c1":
        return scenarios.c1_hill(ncols)
    return scenarios.SCENARIOS[name](ncols, nrows)


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons while the timed region runs."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
    }

    def __init__(self, device: int, period_s: float = 0.01):
        self.samples = []
        self.reasons = 0
        self.period = period_s
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def _sample(self):
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            pass

    def __enter__(self):
        if self.ok:
            self._sample()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()
            self._sample()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        names = [k for k, v in self.REASONS.items() if self.reasons & v and k != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": names, "samples": len(self.samples)}


def cpu_reference(config, ncols, nrows, steps, lanes, timeout=600, stack=1):
    """The reference (oracle/_ref, else the C port) timed on this host, in a child process.
    stack > 1: the weak-scaling grid of `bench.py --gpus stack` (row-stacked copies)."""
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--config", config, "--ncols", str(ncols),
           "--nrows", str(nrows), "--steps", str(steps), "--lanes", str(lanes), "--stack", str(stack)]
    try:
        out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
        line = [l for l in out.stdout.splitlines() if l.startswith("{")]
        if out.returncode == 0 and line:
            r = json.loads(line[-1])
            if lanes > 1 and not r.get("serial_match", True):
                r["note"] = "parallel backend diverged from serial (App. B1); serial timing below"
                raise RuntimeError("mismatch")
            return r
        err = (out.stderr or "")[-300:]
    except Exception as e:  # crash of the racy pool (App. B1) -> serial
        err = str(e)
    if lanes > 1:
        r = cpu_reference(config, ncols, nrows, max(1, steps // 4), 1, timeout, stack)
        r["note"] = f"DataParallel({lanes}) failed ({err.strip()[:120]}); serial backend"
        return r
    raise RuntimeError("CPU reference failed: " + err)


class RunClock:
    """The run loop's output schedule (solver.cpp:627-649): steps are taken toward
    t_next = min(next_out, t_end) and stop on exact output hits, as Simulator::run does."""

    def __init__(self, sim):
        tu = sim.cfg.scaling.t_unit()
        self.sim, self.t = sim, 0.0
        self.t_end = sim.cfg.t_end / tu
        self.dt_out = sim.cfg.dt_out / tu
        self.next_out = self.dt_out

    def advance(self, k):
        done = 0
        while done < k and self.t < self.t_end:
            t_next = min(self.next_out, self.t_end)
            self.t, n, hit = self.sim.steps(self.t, t_next, k - done, t_end=self.t_end)
            done += n
            if hit and t_next == self.next_out:
                self.next_out += self.dt_out
        return done


def time_stages(sim, n=20):
    """Per-stage kernel time in the production context: n steps of the device loop replayed
    from a one-step CUDA graph with events recorded on the launching stream right around
    the predictor and corrector kernels (tp_steps_timed).  Returns mean ms per launch and
    the tiles the last step processed."""
    import ctypes as C
    t = C.c_double(sim._bench_t)
    steps, hit = C.c_long(), C.c_int()
    pm, cm = C.c_float(), C.c_float()
    tu = sim.cfg.scaling.t_unit()
    sim._check(sim.L.tp_steps_timed(sim.h, sim._bench_t_next, sim.cfg.t_end / tu, n, C.byref(t), C.byref(steps),
                                    C.byref(hit), C.byref(pm), C.byref(cm)))
    sim._bench_t = t.value
    k = max(steps.value, 1)
    p_, c_, _ = sim.active_tiles()
    return pm.value / k, cm.value / k, p_, c_


def ncu_traffic():
    """dram bytes per launch of the stage kernels from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_stage_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d


def run_b200(args):
    import torch
    from paper_2104_06784_b200.simulator import Simulator

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2104_06784_b200 import distributed
        return distributed.bench_main(args, METRIC, clock_sampler=ClockSampler)

    torch.cuda.set_device(0)
    sc = scenario_for(args.config, args.ncols, args.nrows)
    cells = sc.ncols * sc.nrows
    t_setup = time.perf_counter()
    sim = Simulator.from_scenario(sc, device=0)
    sim.set_option("graph_steps", args.graph_steps)
    stream = torch.cuda.Stream()
    sim.set_stream(stream.cuda_stream)
    setup_s = time.perf_counter() - t_setup

    clock = RunClock(sim)
    clock.advance(args.warmup)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with clocks:
        torch.cuda.synchronize()
        e0.record(stream)
        n = clock.advance(args.steps)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = sim.kernel_launches()
    act_p, act_c, ntiles = sim.active_tiles()
    assert n == args.steps, (n, args.steps)
    value = cells * args.steps / (ms / 1e3) / 1e9

    # roofline leg: the two stage kernels (the dominant kernel of the step)
    sim._bench_t = clock.t
    sim._bench_t_next = min(clock.next_out, clock.t_end)
    t_pred, t_corr, tp_p, tp_c = time_stages(sim, n=args.roofline_reps)
    peak, peak_src = load_peaks()
    achieved = ALG_BYTES_PER_CELL_UPDATE * cells / ((t_pred + t_corr) / 1e3) / 1e9
    # the same bytes restricted to the tiles the kernels actually processed (dry tiles whose
    # stage is a bitwise no-op are skipped): the kernel's own bandwidth
    frac_p, frac_c = tp_p / ntiles, tp_c / ntiles
    achieved_proc = (ALG_BYTES_PRED * cells * frac_p + ALG_BYTES_CORR * cells * frac_c) / \
        ((t_pred + t_corr) / 1e3) / 1e9
    traffic = None
    nt = ncu_traffic()
    prof = None
    for cand in (nt, (nt or {}).get("wet")):
        if cand and cand.get("grid") == [sc.ncols, sc.nrows] and cand.get("config") == args.config:
            prof = cand
    if prof:
        traffic = prof["dram_bytes_per_step"]
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "stage_kernel<pred>+stage_kernel<corr> per step",
                "alg_bytes_per_launch": ALG_BYTES_PER_CELL_UPDATE * cells,
                "kernel_ms_per_step": round(t_pred + t_corr, 4), "pred_ms": round(t_pred, 4),
                "corr_ms": round(t_corr, 4), "peak_source": peak_src,
                "processed_tile_frac": [round(frac_p, 4), round(frac_c, 4)],
                "achieved_processed_tiles": round(achieved_proc, 1),
                "frac_processed_tiles": round(achieved_proc / peak, 4),
                "step_frac": round(achieved * (t_pred + t_corr) / (ms / args.steps) / peak, 4)}
    if prof and prof.get("fp64_pipe_active_pct"):
        # the processed tiles are FP64-issue bound: the co-bound from the same capture
        roofline["co_bound"] = {"pipe": "fp64", "fp64_pipe_active_pct": prof["fp64_pipe_active_pct"],
                                "issue_active_pct": prof["issue_active_pct"],
                                "dram_throughput_pct": prof["dram_throughput_pct"],
                                "kernels": ["stage_kernel<pred>", "stage_kernel<corr>"],
                                "source": nt.get("source")}

    # e2e leg: through the C ABI with HOST (pinned) buffers, copies inside the timed region
    import ctypes as C
    nbytes = 6 * sim.ny * sim.nx * 8
    h_in = torch.empty(6 * sim.ny * sim.nx, dtype=torch.float64, pin_memory=True)
    h_out = torch.empty_like(h_in, pin_memory=True)  # empty_like alone is pageable
    assert h_in.is_pinned() and h_out.is_pinned()
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h_in.data_ptr(), C.POINTER(C.c_double))))
    # first DMA into a freshly pinned buffer pays ~80 ms of page setup: touch h_out at setup
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), C.POINTER(C.c_double))))
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    sim._check(sim.L.tp_set_state(sim.h, C.cast(h_in.data_ptr(), C.POINTER(C.c_double))))
    clock.t = sim._bench_t
    while clock.next_out <= clock.t:  # an output hit inside the roofline leg
        clock.next_out += clock.dt_out
    ne = clock.advance(args.steps)
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), C.POINTER(C.c_double))))
    w1 = time.perf_counter()
    e2e = {"value": round(cells * ne / (w1 - w0) / 1e9, 4), "unit": "GCUPS",
           "h2d_bytes_per_step": nbytes // max(ne, 1), "d2h_bytes_per_step": nbytes // max(ne, 1),
           "mode": f"tp_set_state(pinned host) + tp_steps({ne}) + tp_get_state(pinned host), wall clock"}

    cpu = None
    if not args.no_cpu:
        lanes = os.cpu_count() or 1
        c = cpu_reference(args.config, sc.ncols, sc.nrows, args.cpu_steps, lanes)
        cpu = {"value": round(c["value"] / 1e9, 6), "unit": "GCUPS", "cores": c["lanes"],
               "kind": "reference" if c["kind"] == "ref" else "port",
               "sample": f"{c['steps']} steps of the same {sc.ncols}x{sc.nrows} {args.config} workload "
                         f"from t=0 (after 1 untimed step), BackendConfig::"
                         f"{'parallel(%d)' % c['lanes'] if c['lanes'] > 1 else 'serial()'}",
               "seconds": round(c["seconds"], 3)}
        if "note" in c:
            cpu["note"] = c["note"]

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "GCUPS", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (deterministic {sc.name} generator in scenarios.py: DEM + "
                f"{'inflow hydrograph' if sc.config.inflow else 'compact release'}; no network data)",
        "config": {"workload": f"{sc.name} {'Mode-II inflow' if sc.config.inflow else 'Mode-I release'}, "
                               f"{sc.ncols}x{sc.nrows} interior cells, cellsize {sc.cellsize:g} m, Table-1 "
                               f"parameters, CFL {sc.config.cfl:g}, output every {sc.config.dt_out:g} s",
                   "grid": [sc.ncols, sc.nrows], "wet_fraction_t0": round(float((sc.h0 > 0).mean()), 4)
                   if sc.h0 is not None else None,
                   "l2": "inputs larger than L2 (state 2x%.0f MB + geometry %.0f MB > 126 MB)"
                         % (nbytes / 1e6, 18 * sim.ny * sim.nx * 8 / 1e6),
                   "parallelism": "single device", "graph_steps": args.graph_steps,
                   "active_tiles_last_step": [act_p, act_c, ntiles],
                   "hbm_roofline_gcups": round(peak / ALG_BYTES_PER_CELL_UPDATE, 3),
                   "hbm_frac_of_step": round(value / (peak / ALG_BYTES_PER_CELL_UPDATE), 4),
                   "setup_seconds": round(setup_s, 2)},
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clocks.summary(), "gpu_launches": launches,
    }
    print(json.dumps(out))


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on this host's cores, on the
    grid our arm runs at this N (N=1: the config's grid; N>1: the weak-scaling grid of N
    row-stacked copies, distributed.bench_main).  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    sc = scenario_for(args.config, args.ncols, args.nrows)
    if world > 1:
        from paper_2104_06784_b200 import scenarios
        sc = (scenarios.SCENARIOS["c3"](args.ncols, args.nrows * world) if args.config == "c3"
              else scenarios.stacked(sc, world))
    lanes = os.cpu_count() or 1
    # bounded sample: at most ~2 minutes of CPU work
    steps = args.steps
    probe = cpu_reference(args.config, args.ncols, args.nrows, 1, lanes, stack=world)
    per_step = probe["seconds"] / max(probe["steps"], 1)
    if per_step * steps > 120:
        steps = max(1, int(120 / per_step))
    c = cpu_reference(args.config, args.ncols, args.nrows, steps, lanes, stack=world)
    assert c["grid"] == [sc.ncols, sc.nrows], (c["grid"], sc.ncols, sc.nrows)
    v = round(c["value"] / 1e9, 6)
    cpu = {"value": v, "unit": "GCUPS", "cores": c["lanes"],
           "kind": "reference" if c["kind"] == "ref" else "port",
           "sample": f"{c['steps']} steps of {sc.ncols}x{sc.nrows} {args.config} (of {args.steps} requested)"}
    if "note" in c:
        cpu["note"] = c["note"]
    out = {"metric": METRIC, "value": v, "unit": "GCUPS", "n_gpus": args.gpus, "steps": c["steps"],
           "warmup": args.warmup, "ms_per_step": round(1e3 * c["seconds"] / c["steps"], 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (scenarios.py)", "impl": "reference",
           "config": {"workload": f"{sc.name} {sc.ncols}x{sc.nrows}", "grid": [sc.ncols, sc.nrows],
                      "parallelism": f"host CPU, {c['lanes']} threads"},
           "cpu_baseline": cpu, "e2e": {"value": v, "unit": "GCUPS", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "wet"])
    ap.add_argument("--ncols", type=int, default=2048)
    ap.add_argument("--nrows", type=int, default=2048)
    ap.add_argument("--graph-steps", type=int, default=16)
    ap.add_argument("--roofline-reps", type=int, default=20)
    ap.add_argument("--cpu-steps", type=int, default=60)  # ~10 s of the reference on 16 cores at C2
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
