import sys, os, time, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.simulator import Simulator
sc = scenarios.c2_valley(2048, 2048)
sim = Simulator.from_scenario(sc)
sim.steps(0.0, 1e9, 5, t_end=1e9)
n = 6 * sim.ny * sim.nx
h = torch.empty(n, dtype=torch.float64, pin_memory=True)
dp = C.POINTER(C.c_double)
for k in range(4):
    t0 = time.perf_counter()
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h.data_ptr(), dp)))
    t1 = time.perf_counter()
    print(f"tp_get_state {1e3*(t1-t0):.2f} ms  {n*8/(t1-t0)/1e9:.1f} GB/s")
import numpy as np
a = np.empty(n)
for k in range(2):
    t0 = time.perf_counter()
    sim._check(sim.L.tp_get_state(sim.h, a.ctypes.data_as(dp)))
    t1 = time.perf_counter()
    print(f"tp_get_state (pageable numpy) {1e3*(t1-t0):.2f} ms")
