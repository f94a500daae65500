"""Quick device timing of tp_steps on a scenario (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.simulator import Simulator

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fastdiv = int(sys.argv[4]) if len(sys.argv) > 4 else 1
gs = int(sys.argv[5]) if len(sys.argv) > 5 else 16
sc = scenarios.SCENARIOS[name](n, n) if name != "c1" else scenarios.c1_hill(n)
t0 = time.time()
sim = Simulator.from_scenario(sc, fastdiv=bool(fastdiv))
sim.set_option("graph_steps", gs)
import os
print(f"setup {time.time()-t0:.2f}s  grid {sc.ncols}x{sc.nrows} wet frac {np.mean(sc.h0 > 0) if sc.h0 is not None else 0:.3f}")
t, n_, hit = sim.steps(0.0, 1e9, 8, t_end=1e9)   # warmup
sim.synchronize()
t1 = time.perf_counter()
t, n_, hit = sim.steps(t, 1e9, steps, t_end=1e9)
sim.synchronize()
t2 = time.perf_counter()
cu = sc.ncols * sc.nrows * n_ / (t2 - t1) if n_ else 0.0
print(f"{name} {sc.ncols}x{sc.nrows} fastdiv={fastdiv} steps={n_} {1e3*(t2-t1)/max(n_, 1):.3f} ms/step  {cu/1e9:.3f} GCUPS  "
      f"HBM-frac {cu*464/6449.1e9:.3f}  launches={sim.kernel_launches()}")
