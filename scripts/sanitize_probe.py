"""Small device-loop + step-piece run for compute-sanitizer (memcheck / racecheck / synccheck).
Usage: compute-sanitizer --tool racecheck python scripts/sanitize_probe.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2104_06784_b200 import scenarios  # noqa: E402
from paper_2104_06784_b200.simulator import Simulator  # noqa: E402

for sc, wide in ((scenarios.c1_hill(40), 0), (scenarios.wet_valley(37, 33), 0),
                 (scenarios.c3_channel(48, 32, t_end=30.0, dt_out=0.5), 0),
                 (scenarios.c1_hill(40), 1 << 30), (scenarios.wet_valley(37, 33), 1 << 30)):
    sim = Simulator.from_scenario(sc)
    sim.set_option("wide_tiles", wide)  # production (2 CTAs/SM) and wide (512-thread) stage CTAs
    if sc.config.inflow:  # Mode-II: several output intervals (inflow-window checks, safe inflow tiles)
        t, n = 0.0, 0
        for k in range(1, 5):
            t, nk, _ = sim.steps(t, k * 0.5 / sc.config.scaling.t_unit(), 6, t_end=1e9)
            n += nk
    else:
        t, n, _ = sim.steps(0.0, 1e9, 6, t_end=1e9)
    sim.apply_boundaries(t)
    dt = sim.compute_dt(t, 1e9)
    sim.advance_step(dt, t)
    sim.regularize()
    s = sim.state()
    sim.snapshot(t)
    sim.interior_mass_device()
    assert np.isfinite(s).all()
    print(sc.name, "ok", n)

# peer-joined slabs on one device (in-kernel halo wait, back-region tiles), both CTA shapes
import torch  # noqa: E402
from paper_2104_06784_b200.distributed import CudaSlab, PeerGroup, decompose  # noqa: E402
for wide in (0, 1 << 30):
    sc = scenarios.c1_hill(64)
    slabs = [CudaSlab(sc, r, stream=torch.cuda.Stream()) for r in decompose(sc.nrows, 3)]
    for sl in slabs:
        sl.sim.set_option("wide_tiles", wide)
    t, n, _ = PeerGroup(slabs).steps(0.0, 1e9, 6, t_end=1e9)
    print("peer group", "wide" if wide else "dense", "ok", n)
