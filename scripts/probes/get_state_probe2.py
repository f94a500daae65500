"""Where does tp_get_state's time go: library D2H into torch-pinned vs pageable memory, and
torch's own D2H into the same pinned buffer."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_06784_b200 import scenarios  # noqa: E402
from paper_2104_06784_b200.simulator import Simulator  # noqa: E402

sc = scenarios.c2_valley(2048, 2048)
sim = Simulator.from_scenario(sc)
sim.steps(0.0, 1e9, 4, t_end=1e9)
n = 6 * sim.ny * sim.nx
dp = C.POINTER(C.c_double)
h_pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_np = np.empty(n)
d = torch.randn(n, dtype=torch.float64, device="cuda")
for what, ptr in (("pinned", h_pin.data_ptr()), ("pageable", h_np.ctypes.data)):
    for rep in range(3):
        t0 = time.perf_counter()
        sim._check(sim.L.tp_get_state(sim.h, C.cast(ptr, dp)))
        t1 = time.perf_counter()
        sim._check(sim.L.tp_set_state(sim.h, C.cast(ptr, dp)))
        t2 = time.perf_counter()
    print(f"{what}: get {1e3 * (t1 - t0):.1f} ms  set {1e3 * (t2 - t1):.1f} ms")
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h_pin.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
print(f"torch D2H into the same pinned buffer {1e3 * (t1 - t0):.1f} ms")
