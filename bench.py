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


def cpu_reference(config, ncols, nrows, steps, lanes, timeout=600, stack=1, check_serial=1):
    """The reference (oracle/_ref, else the C port) timed on this host, in a child process.
    stack > 1: the weak-scaling grid of `bench.py --gpus stack` (row-stacked copies).
    check_serial: steps of a serial run the parallel state must match bitwise (App. B1)."""
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--config", config, "--ncols", str(ncols),
           "--nrows", str(nrows), "--steps", str(steps), "--lanes", str(lanes), "--stack", str(stack),
           "--check-serial", str(check_serial)]
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
        r = cpu_reference(config, ncols, nrows, max(1, steps // 4), 1, timeout, stack, 0)
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
        self.steps = 0  # steps taken through this clock

    def advance(self, k):
        done = 0
        while done < k and self.t < self.t_end:
            t_next = min(self.next_out, self.t_end)
            self.t, n, hit = self.sim.steps(self.t, t_next, k - done, t_end=self.t_end)
            done += n
            if hit and t_next == self.next_out:
                self.next_out += self.dt_out
        self.steps += done
        return done


def time_stages(sim, n=20):
    """Per-stage kernel time in the production context: n steps of the device loop replayed
    from a one-step CUDA graph with events recorded on the launching stream right around
    the predictor and corrector kernels (tp_steps_timed).  Returns mean ms per launch and
    the mean tiles per launch the two stages processed over those steps."""
    import ctypes as C
    t = C.c_double(sim._bench_t)
    steps, hit = C.c_long(), C.c_int()
    pm, cm = C.c_float(), C.c_float()
    tu = sim.cfg.scaling.t_unit()
    sim._check(sim.L.tp_steps_timed(sim.h, sim._bench_t_next, sim.cfg.t_end / tu, n, C.byref(t), C.byref(steps),
                                    C.byref(hit), C.byref(pm), C.byref(cm)))
    sim._bench_t = t.value
    k = max(steps.value, 1)
    tp_, tc_ = C.c_longlong(), C.c_longlong()
    sim._check(sim.L.tp_timed_tiles(sim.h, C.byref(tp_), C.byref(tc_)))
    sim._bench_steps = steps.value
    return pm.value / k, cm.value / k, tp_.value / k, tc_.value / k


def ncu_traffic():
    """dram bytes per launch of the stage kernels from the committed ncu summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_stage_summary.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    return d


def workload_config(sc) -> dict:
    """The `config` keys both arms print for a scenario (identical strings, so the driver
    can match the reference arm's line to ours)."""
    return {"workload": f"{sc.name} {'Mode-II inflow' if sc.config.inflow else 'Mode-I release'}, "
                        f"{sc.ncols}x{sc.nrows} interior cells, cellsize {sc.cellsize:g} m, Table-1 "
                        f"parameters, CFL {sc.config.cfl:g}, output every {sc.config.dt_out:g} s",
            "grid": [sc.ncols, sc.nrows]}


def wet_fraction(sim) -> float:
    """Fraction of interior cells with a nonzero thickness (state downloaded once)."""
    s = sim.state()
    h = s[0, 3:-3, 3:-3] + s[1, 3:-3, 3:-3]
    return float((h != 0.0).mean())


def timed_steps(sim, clock, stream, steps):
    """CUDA-event time (ms) of `steps` device-loop steps along the run schedule."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    n = clock.advance(steps)
    e1.record(stream)
    torch.cuda.synchronize()
    assert n == steps, (n, steps)
    return e0.elapsed_time(e1)


def stage_roofline(sim, clock, cells, reps, peak):
    """Roofline of the dominant kernel (the two stage kernels of a step), timed in the
    production context (tp_steps_timed: CUDA events on the launching stream around each
    stage kernel of a one-step graph, `reps` steps).  `achieved` counts the algorithmic
    bytes (208 B predictor + 256 B corrector per cell-update) of the tiles
    the kernels processed (dry tiles whose stage is a bitwise no-op are not read, DESIGN.md
    §3); `effective_*` counts every interior cell as updated."""
    sim._bench_t = clock.t
    sim._bench_t_next = min(clock.next_out, clock.t_end)
    t_pred, t_corr, tp_p, tp_c = time_stages(sim, n=reps)
    clock.t = sim._bench_t
    clock.steps += sim._bench_steps
    while clock.next_out <= clock.t:  # an output hit inside this leg
        clock.next_out += clock.dt_out
    _, _, ntiles = sim.active_tiles()
    frac_p, frac_c = tp_p / ntiles, tp_c / ntiles
    kms = t_pred + t_corr
    alg_proc = ALG_BYTES_PRED * cells * frac_p + ALG_BYTES_CORR * cells * frac_c
    achieved = alg_proc / (kms / 1e3) / 1e9
    eff = ALG_BYTES_PER_CELL_UPDATE * cells / (kms / 1e3) / 1e9
    return {"achieved": round(achieved, 1), "frac": round(achieved / peak, 4),
            "alg_bytes_per_step": int(alg_proc), "kernel_ms_per_step": round(kms, 4),
            "pred_ms": round(t_pred, 4), "corr_ms": round(t_corr, 4),
            "processed_tile_frac": [round(frac_p, 4), round(frac_c, 4)],
            "effective_achieved": round(eff, 1), "effective_frac": round(eff / peak, 4)}


def make_sim(sc, graph_steps):
    import torch
    from paper_2104_06784_b200.simulator import Simulator
    t0 = time.perf_counter()
    sim = Simulator.from_scenario(sc, device=0)
    sim.set_option("graph_steps", graph_steps)
    stream = torch.cuda.Stream()
    sim.set_stream(stream.cuda_stream)
    return sim, stream, time.perf_counter() - t0


def run_b200(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or args.gpus > 1:
        from paper_2104_06784_b200 import distributed
        return distributed.bench_main(args, METRIC, clock_sampler=ClockSampler)

    torch.cuda.set_device(0)
    peak, peak_src = load_peaks()
    sc = scenario_for(args.config, args.ncols, args.nrows)
    cells = sc.ncols * sc.nrows
    sim, stream, setup_s = make_sim(sc, args.graph_steps)

    clock = RunClock(sim)
    clock.advance(args.warmup)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    with clocks:
        ms = timed_steps(sim, clock, stream, args.steps)
    launches = sim.kernel_launches()
    act_p, act_c, ntiles = sim.active_tiles()
    value = cells * args.steps / (ms / 1e3) / 1e9

    # roofline leg: the two stage kernels (the dominant kernel of the step)
    rl = stage_roofline(sim, clock, cells, args.roofline_reps, peak)
    traffic = None
    nt = ncu_traffic()
    prof = None
    for cand in (nt, (nt or {}).get("wet")):
        if cand and cand.get("grid") == [sc.ncols, sc.nrows] and cand.get("config") == args.config:
            prof = cand
    if prof:
        traffic = prof["dram_bytes_per_step"]
    roofline = {"bound": "hbm", "achieved": rl["achieved"], "peak": peak, "unit": "GB/s",
                "frac": rl["frac"], "traffic": traffic,
                "kernel": "stage_kernel<pred>+stage_kernel<corr> per step (achieved: algorithmic "
                          "bytes of the processed tiles / their CUDA-event time)",
                "peak_source": peak_src}
    roofline.update({k: v for k, v in rl.items() if k not in ("achieved", "frac")})
    roofline["step_frac"] = round(rl["frac"] * rl["kernel_ms_per_step"] / (ms / args.steps), 4)
    if prof and prof.get("fp64_pipe_active_pct"):
        # the processed tiles are FP64-issue bound: the co-bound from the same capture
        roofline["co_bound"] = {"pipe": "fp64", "fp64_pipe_active_pct": prof["fp64_pipe_active_pct"],
                                "issue_active_pct": prof["issue_active_pct"],
                                "dram_throughput_pct": prof["dram_throughput_pct"],
                                "kernels": ["stage_kernel<pred>", "stage_kernel<corr>"],
                                "source": nt.get("source")}
        ir = nt.get("instruction_roofline")
        if ir:
            # the processed tiles against the instruction ceilings of the same code: the FP64
            # pipe (64 thread ops per clock per SM) and issue (128 thread instructions per
            # clock per SM) at the measured instruction counts per cell-update
            rate = roofline["achieved"] * 1e9 / ALG_BYTES_PER_CELL_UPDATE / 1e9  # processed GCUPS
            roofline["co_bound"].update({
                "fp64_thread_ops_per_cell_update": ir["fp64_thread_ops_per_cell_update"],
                "thread_instructions_per_cell_update": ir["thread_instructions_per_cell_update"],
                "fp64_ceiling_gcups": ir["fp64_ceiling_gcups"], "issue_ceiling_gcups": ir["issue_ceiling_gcups"],
                "processed_gcups": round(rate, 3),
                "frac_of_issue_ceiling": round(rate / ir["issue_ceiling_gcups"], 4)})

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
    ne = clock.advance(args.steps)
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), C.POINTER(C.c_double))))
    w1 = time.perf_counter()
    e2e = {"value": round(cells * ne / (w1 - w0) / 1e9, 4), "unit": "GCUPS",
           "h2d_bytes_per_step": nbytes // max(ne, 1), "d2h_bytes_per_step": nbytes // max(ne, 1),
           "mode": f"tp_set_state(pinned host) + tp_steps({ne}) + tp_get_state(pinned host), wall clock"}
    del h_in, h_out

    extra = {}
    if not args.no_extra:
        # a representative window of a whole run: after the release has spread
        extra["long_run"] = long_run_leg(sim, clock, stream, cells, peak, args)
        sim.close()
        del sim
        torch.cuda.empty_cache()
        # the north-star grid (BASELINE.json configs[4]): C5 8192^2, N=1
        extra["c5_8192"] = c5_leg(args, peak)
        # the latency-bound sparse steps (the per-step floor): BASELINE.json
        # configs[2] (C3 Mode-II channel) and configs[0] (C1 hill), along their output schedules
        extra["sparse_steps"] = {"c3_4096x2048": sparse_leg("c3", 4096, 2048, 400, args),
                                 "c1_256": sparse_leg("c1", 256, 256, 500, args)}

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

    cfg = workload_config(sc)
    cfg.update({"wet_fraction_t0": round(float((sc.h0 > 0).mean()), 4) if sc.h0 is not None else None,
                "l2": "inputs larger than L2 (state 2x%.0f MB + geometry %.0f MB > 126 MB)"
                      % (nbytes / 1e6, 18 * (nbytes // 48) * 8 / 1e6),
                "parallelism": "single device", "graph_steps": args.graph_steps,
                "window": f"steps {args.warmup + 1}..{args.warmup + args.steps} from t=0",
                "active_tiles_last_step": [act_p, act_c, ntiles],
                "hbm_roofline_gcups": round(peak / ALG_BYTES_PER_CELL_UPDATE, 3),
                "setup_seconds": round(setup_s, 2)})
    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "GCUPS", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": f"synthetic (deterministic {sc.name} generator in scenarios.py: DEM + "
                f"{'inflow hydrograph' if sc.config.inflow else 'compact release'}; no network data)",
        "config": cfg, "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "clocks": clocks.summary(), "gpu_launches": launches,
    }
    out.update(extra)
    print(json.dumps(out))


def long_run_leg(sim, clock, stream, cells, peak, args):
    """GCUPS and the stage kernels' roofline on a window after the release has spread:
    the run continues to step `--long-start`, then `--long-steps` steps are timed; the wet
    fraction (cells with a nonzero thickness) is reported at the window's start and end."""
    while clock.steps < args.long_start:
        if clock.advance(min(args.long_start - clock.steps, 500)) == 0:
            break  # t_end reached
    first = clock.steps + 1
    w0 = wet_fraction(sim)
    ms = timed_steps(sim, clock, stream, args.long_steps)
    w1 = wet_fraction(sim)
    rl = stage_roofline(sim, clock, cells, args.roofline_reps, peak)
    return {"value": round(cells * args.long_steps / (ms / 1e3) / 1e9, 4), "unit": "GCUPS",
            "steps": args.long_steps, "ms_per_step": round(ms / args.long_steps, 5),
            "window": f"steps {first}..{first + args.long_steps - 1} of the same run from t=0 "
                      f"(t = {clock.t * sim.cfg.scaling.t_unit():.2f} s at the end)",
            "wet_fraction": [round(w0, 4), round(w1, 4)],
            "roofline": {"frac": rl["frac"], "achieved": rl["achieved"],
                         "processed_tile_frac": rl["processed_tile_frac"],
                         "effective_frac": rl["effective_frac"]}}


def c5_leg(args, peak):
    """BASELINE.json configs[4] at its smallest point, the north-star grid: the C2 valley
    generator at 8192 x 8192 on one GPU (weak-scaling base case of bench.py --gpus N)."""
    import torch
    sc = scenario_for("c2", args.c5_size, args.c5_size)
    cells = sc.ncols * sc.nrows
    sim, stream, setup_s = make_sim(sc, args.graph_steps)
    clock = RunClock(sim)
    clock.advance(args.warmup)
    torch.cuda.synchronize()
    clocks = ClockSampler(0)
    with clocks:
        ms = timed_steps(sim, clock, stream, args.c5_steps)
    rl = stage_roofline(sim, clock, cells, max(4, args.roofline_reps // 2), peak)
    out = {"value": round(cells * args.c5_steps / (ms / 1e3) / 1e9, 4), "unit": "GCUPS",
           "steps": args.c5_steps, "warmup": args.warmup, "ms_per_step": round(ms / args.c5_steps, 5),
           "config": workload_config(sc), "setup_seconds": round(setup_s, 2),
           "roofline": {"bound": "hbm", "achieved": rl["achieved"], "peak": peak, "unit": "GB/s",
                        "frac": rl["frac"], "traffic": None, **{k: v for k, v in rl.items()
                                                               if k not in ("achieved", "frac")}},
           "clocks": clocks.summary()}
    nt = ncu_traffic()
    c5p = (nt or {}).get("c5")
    if c5p and c5p.get("grid") == [sc.ncols, sc.nrows]:
        out["roofline"]["traffic"] = c5p["dram_bytes_per_step"]
        out["roofline"]["traffic_source"] = nt.get("source")
    sim.close()
    del sim
    torch.cuda.empty_cache()
    return out


def sparse_leg(config, ncols, nrows, steps, args):
    """ms per step of a latency-bound workload (a few dozen listed tiles per stage) along its
    run's output schedule, after 10 untimed steps; CUDA events on the launching stream."""
    import torch
    sc = scenario_for(config, ncols, nrows)
    sim, stream, _ = make_sim(sc, args.graph_steps)
    clock = RunClock(sim)
    clock.advance(10)
    torch.cuda.synchronize()
    ms = timed_steps(sim, clock, stream, steps)
    act = sim.active_tiles()
    out = {"ms_per_step": round(ms / steps, 5), "steps": steps,
           "value": round(sc.ncols * sc.nrows * steps / (ms / 1e3) / 1e9, 4), "unit": "GCUPS",
           "tiles_listed_last_step": [act[0], act[1]], "tiles": act[2],
           "workload": workload_config(sc)["workload"]}
    sim.close()
    del sim
    torch.cuda.empty_cache()
    return out


def run_reference(args):
    """--impl reference: the reference's own CPU implementation on this host's cores, on the
    grid our arm runs at this N (N=1: the config's grid; N>1: the grid of distributed.bench_main,
    weak: N row-stacked copies, strong: the one grid).  Under torchrun only rank 0 runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = max(args.gpus, int(os.environ.get("WORLD_SIZE", "1")))
    from paper_2104_06784_b200 import distributed
    sc, stack = distributed.bench_scenario(args, world) if world > 1 else \
        (scenario_for(args.config, args.ncols, args.nrows), 1)
    lanes = os.cpu_count() or 1
    # bounded sample: at most ~2 minutes of CPU work
    steps = args.steps
    probe = cpu_reference(args.config, args.ncols, args.nrows, 1, lanes, stack=stack)
    per_step = probe["seconds"] / max(probe["steps"], 1)
    if per_step * steps > 120:
        steps = max(1, int(120 / per_step))
    c = cpu_reference(args.config, args.ncols, args.nrows, steps, lanes, stack=stack)
    assert c["grid"] == [sc.ncols, sc.nrows], (c["grid"], sc.ncols, sc.nrows)
    v = round(c["value"] / 1e9, 6)
    cpu = {"value": v, "unit": "GCUPS", "cores": c["lanes"],
           "kind": "reference" if c["kind"] == "ref" else "port",
           "sample": f"{c['steps']} steps of {sc.ncols}x{sc.nrows} {args.config} (of {args.steps} requested)"}
    if "note" in c:
        cpu["note"] = c["note"]
    cfg = workload_config(sc)
    cfg["parallelism"] = f"host CPU, {c['lanes']} threads"
    out = {"metric": METRIC, "value": v, "unit": "GCUPS", "n_gpus": args.gpus, "steps": c["steps"],
           "warmup": args.warmup, "ms_per_step": round(1e3 * c["seconds"] / c["steps"], 3),
           "higher_is_better": True, "scaling": "strong" if getattr(args, "scaling", "weak") == "strong" else "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic (scenarios.py)", "impl": "reference",
           "config": cfg,
           "cpu_baseline": cpu, "e2e": {"value": v, "unit": "GCUPS", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}
    if world == 1 and not args.no_extra:
        # the north-star grid beside it (our arm's c5_8192 object): a 2-step sample
        try:
            # (the parallel-vs-serial bitwise check runs on the 2048^2 line; a serial 8192^2
            # step alone takes about a minute)
            c5 = cpu_reference("c2", args.c5_size, args.c5_size, args.c5_ref_steps, lanes, timeout=900,
                               check_serial=0)
            out["c5_8192"] = {"value": round(c5["value"] / 1e9, 6), "unit": "GCUPS",
                              "steps": c5["steps"], "ms_per_step": round(1e3 * c5["seconds"] / c5["steps"], 3),
                              "config": workload_config(scenario_for("c2", args.c5_size, args.c5_size)),
                              "cores": c5["lanes"], "setup_seconds": round(c5.get("setup_seconds", 0.0), 1)}
        except Exception as e:  # noqa: BLE001 - a reported gap, not a failed arm
            out["c5_8192"] = {"unavailable": str(e)[:200]}
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
    ap.add_argument("--no-extra", action="store_true", help="skip the long-run window and the C5 8192^2 leg")
    ap.add_argument("--long-start", type=int, default=1000)
    ap.add_argument("--long-steps", type=int, default=200)
    ap.add_argument("--c5-size", type=int, default=8192)
    ap.add_argument("--c5-steps", type=int, default=20)
    ap.add_argument("--c5-ref-steps", type=int, default=2)
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="N>1: weak = one copy of the N=1 workload per GPU; strong = one grid split N ways")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
