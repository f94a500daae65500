"""TEST INFRASTRUCTURE ONLY — CPU timing of the reference implementation.

Runs in its own process (the reference's DataParallel backend has a dispatch
race that can crash on some workloads), on a bounded sample
of a bench workload: the UNMODIFIED reference compiled in place (oracle/_ref,
``kind=ref``) or, where /root/reference was absent at build time, the C
restatement (``kind=port``).  Prints one JSON line.

  python -m oracle.cpu_bench --config c2 --ncols 2048 --nrows 2048 --steps 6 --lanes 16
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--ncols", type=int, default=2048)
    ap.add_argument("--nrows", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--lanes", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--kind", default="auto")
    ap.add_argument("--stack", type=int, default=1,
                    help="weak-scaling grid of bench.py --gpus N: N row-stacked copies (C3: N x the rows)")
    ap.add_argument("--check-serial", type=int, default=1,
                    help="steps of a serial run the parallel state must match bitwise (App. B1)")
    a = ap.parse_args()

    import numpy as np
    from oracle import oracle as orc
    from paper_2104_06784_b200 import scenarios

    kind = a.kind
    if kind == "auto":
        kind = "ref" if (orc.available("ref") or os.path.exists(orc.REF_SOURCES)) else "port"
    if a.config == "c1":
        sc = scenarios.c1_hill(a.ncols)
    elif a.config == "c3":
        sc = scenarios.SCENARIOS["c3"](a.ncols, a.nrows * a.stack)
    else:
        sc = scenarios.SCENARIOS[a.config](a.ncols, a.nrows)
    if a.stack > 1 and a.config != "c3":
        sc = scenarios.stacked(sc, a.stack)
    lanes = max(1, a.lanes)
    t0 = time.perf_counter()
    sim = orc.OracleSim(sc, kind, lanes=lanes if lanes > 1 else 0)
    setup = time.perf_counter() - t0
    # the run loop's output schedule (solver.cpp:627-649), as bench.py's RunClock: steps go
    # toward min(next output, t_end) and stop on exact hits (a dry Mode-II start jumps to the
    # first output time in one step)
    tu = sc.config.scaling.t_unit()
    t_end, dt_out = sc.config.t_end / tu, sc.config.dt_out / tu
    clock = {"t": 0.0, "next": dt_out}

    def advance(k):
        done = 0
        while done < k and clock["t"] < t_end:
            t_next = min(clock["next"], t_end)
            clock["t"], d, hit = sim.steps(clock["t"], t_next, k - done, t_end=t_end)
            done += len(d)
            if hit and t_next == clock["next"]:
                clock["next"] += dt_out
        return done

    # one untimed step (first-touch of the buffers), then the timed sample
    advance(1)
    t1 = time.perf_counter()
    n = advance(a.steps)
    dt_wall = time.perf_counter() - t1
    out = {"kind": kind, "lanes": lanes, "steps": n, "seconds": dt_wall, "setup_seconds": setup,
           "cells": sc.ncols * sc.nrows, "value": sc.ncols * sc.nrows * n / dt_wall,
           "unit": "cell-updates/s", "config": a.config, "grid": [sc.ncols, sc.nrows]}
    del sim  # (8192^2: ~30 GB of host memory per instance)
    if lanes > 1 and a.check_serial > 0:
        # App. B1: multi-lane timings only count when they match the serial backend bitwise
        par = orc.OracleSim(sc, kind, lanes=lanes)
        ser = orc.OracleSim(sc, kind, lanes=0)
        par.steps(0.0, min(dt_out, t_end), a.check_serial, t_end=t_end)
        ser.steps(0.0, min(dt_out, t_end), a.check_serial, t_end=t_end)
        out["serial_match"] = bool(np.array_equal(par.state().view(np.uint64), ser.state().view(np.uint64)))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
