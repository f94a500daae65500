"""Active / safe tile counts along the run loop's output schedule (development probe).
usage: safe_probe_run.py cfg ncols nrows steps"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_06784_b200 import scenarios  # noqa: E402
from paper_2104_06784_b200.simulator import Simulator  # noqa: E402

name, nc, nr, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
sc = scenarios.SCENARIOS[name](nc, nr)
sim = Simulator.from_scenario(sc)
tu = sc.config.scaling.t_unit()
t_end, dt_out = sc.config.t_end / tu, sc.config.dt_out / tu
t, done, k = 0.0, 0, 1
while done < steps and t < t_end:
    t_next = min(k * dt_out, t_end)
    t, n, hit = sim.steps(t, t_next, min(20, steps - done), t_end=t_end)
    done += n
    if hit:
        k += 1
    p, c, tot = sim.active_tiles()
    print(f"step {done} t={t * tu:.2f}s: active {c}/{tot} safe {sim.safe_tiles()}")
if os.environ.get("VALUE_HIST"):
    import numpy as np
    s = sim.state()[:, 3:-3, 3:-3]
    a = np.abs(s[s != 0.0])
    print("nonzero values", a.size, "negative thickness", int((s[0:2] < 0).sum()))
    for e in (-1000, -800, -300, -100, -30):
        print(f"  |x| < 2^{e}: {(a < 2.0 ** e).sum()}")
    h = sim.state()[0:2, 3:-3, 3:-3]
    print("thickness nonzero < 1e-10 (h_dry):", int(((h > 0) & (h < 1e-10)).sum()), "of", int((h > 0).sum()))
