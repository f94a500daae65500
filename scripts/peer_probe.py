"""PeerGroup of N in-process slabs vs one domain on one GPU: step time, listed tiles and
kTileCond skips (development probe).  usage: peer_probe.py n ncols rows_per steps"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2104_06784_b200 import scenarios  # noqa: E402
from paper_2104_06784_b200.distributed import CudaSlab, PeerGroup, decompose  # noqa: E402
from paper_2104_06784_b200.simulator import Simulator  # noqa: E402

n, nc, rp, steps = (int(a) for a in sys.argv[1:5])
sc = scenarios.stacked(scenarios.c2_valley(nc, rp), n)
one = Simulator.from_scenario(sc)
one.steps(0.0, 1e9, 5, t_end=1e9)
one.synchronize()
t0 = time.perf_counter()
one.steps(1e-9, 1e9, steps, t_end=1e9)
one.synchronize()
t_one = (time.perf_counter() - t0) / steps
print(f"one domain {sc.ncols}x{sc.nrows}: {1e3 * t_one:.3f} ms/step, listed {one.active_tiles()}")
one.close()
slabs = [CudaSlab(sc, r, stream=torch.cuda.Stream()) for r in decompose(sc.nrows, n)]
g = PeerGroup(slabs)
t, _, _ = g.steps(0.0, 1e9, 5, t_end=1e9)
torch.cuda.synchronize()
t0 = time.perf_counter()
g.steps(t, 1e9, steps, t_end=1e9)
torch.cuda.synchronize()
t_grp = (time.perf_counter() - t0) / steps
for s in slabs:
    k = C.c_ulonglong()
    s.sim._check(s.L.tp_cond_skipped_tiles(s.h, C.byref(k)))
    print(f"  slab rows {s.row0}-{s.row1}: listed {s.sim.active_tiles()}, cond skipped {k.value}")
print(f"{n} peer slabs: {1e3 * t_grp:.3f} ms/step")
