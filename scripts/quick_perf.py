"""Quick device timing of tp_steps on a scenario along its output schedule (development aid).
usage: quick_perf.py name [n] [steps] [fastdiv] [graph_steps]   (c3: n x n/2)"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.simulator import Simulator
from bench import RunClock

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fastdiv = int(sys.argv[4]) if len(sys.argv) > 4 else 1
gs = int(sys.argv[5]) if len(sys.argv) > 5 else 16
sc = scenarios.c1_hill(n) if name == "c1" else scenarios.SCENARIOS[name](n, n // 2 if name == "c3" else n)
t0 = time.time()
sim = Simulator.from_scenario(sc, fastdiv=bool(fastdiv))
sim.set_option("graph_steps", gs)
for kv in os.environ.get("QP_OPTS", "").split():  # e.g. QP_OPTS="merge_post=0 wide_tiles=0"
    k, v = kv.split("=")
    sim.set_option(k, int(v))
print(f"setup {time.time()-t0:.2f}s  grid {sc.ncols}x{sc.nrows} wet frac {np.mean(sc.h0 > 0) if sc.h0 is not None else 0:.3f}")
clk = RunClock(sim)
clk.advance(8)  # warmup
out0 = clk.next_out
sim.synchronize()
t1 = time.perf_counter()
n_ = clk.advance(steps)
sim.synchronize()
t2 = time.perf_counter()
cu = sc.ncols * sc.nrows * n_ / (t2 - t1) if n_ else 0.0
print(f"{name} {sc.ncols}x{sc.nrows} fastdiv={fastdiv} steps={n_} {1e3*(t2-t1)/max(n_, 1):.4f} ms/step  {cu/1e9:.3f} GCUPS  "
      f"HBM-frac {cu*464/6557.8e9:.3f}  launches={sim.kernel_launches()}  outputs={round((clk.next_out - out0) / clk.dt_out)}  gs={gs}")
