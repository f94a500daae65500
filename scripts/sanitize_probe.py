"""Small device-loop + step-piece run for compute-sanitizer (memcheck / racecheck / synccheck).
Usage: compute-sanitizer --tool racecheck python scripts/sanitize_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2104_06784_b200 import scenarios  # noqa: E402
from paper_2104_06784_b200.simulator import Simulator  # noqa: E402

for sc in (scenarios.c1_hill(40), scenarios.wet_valley(37, 33),
           scenarios.c3_channel(48, 32, t_end=30.0, dt_out=0.5)):
    sim = Simulator.from_scenario(sc)
    tn = 0.5 / sc.config.scaling.t_unit() if sc.config.inflow else 1e9
    t, n, _ = sim.steps(0.0, tn, 6, t_end=1e9)
    sim.apply_boundaries(t)
    dt = sim.compute_dt(t, 1e9)
    sim.advance_step(dt, t)
    sim.regularize()
    s = sim.state()
    sim.snapshot(t)
    sim.interior_mass_device()
    assert np.isfinite(s).all()
    print(sc.name, "ok", n)
