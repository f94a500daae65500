import sys, time, ctypes as C
sys.path.insert(0, '.')
import torch
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.simulator import Simulator
sc = scenarios.c2_valley(2048, 2048)
sim = Simulator.from_scenario(sc)
t, n, _ = sim.steps(0.0, 1e9, 10, t_end=1e9); sim.synchronize()
h_in = torch.empty(6 * sim.ny * sim.nx, dtype=torch.float64, pin_memory=True)
h_out = torch.empty_like(h_in, pin_memory=True)
dp = C.POINTER(C.c_double)
sim._check(sim.L.tp_get_state(sim.h, C.cast(h_in.data_ptr(), dp)))
t0 = time.perf_counter(); sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), dp))); print(f'warm get into h_out {1e3*(time.perf_counter()-t0):.1f} ms')
for rep in range(3):
    t0 = time.perf_counter()
    sim._check(sim.L.tp_set_state(sim.h, C.cast(h_in.data_ptr(), dp)))
    t1 = time.perf_counter()
    t, n, _ = sim.steps(t, 1e9, 200, t_end=1e9)
    t2 = time.perf_counter()
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), dp)))
    t3 = time.perf_counter()
    print(f"set {1e3*(t1-t0):.1f} ms  steps {1e3*(t2-t1):.1f} ms  get {1e3*(t3-t2):.1f} ms")
sim.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), dp)))
    t1 = time.perf_counter()
    print(f"back-to-back get {1e3*(t1-t0):.1f} ms")
t, n, _ = sim.steps(t, 1e9, 50, t_end=1e9)
t0 = time.perf_counter(); sim.synchronize(); t1 = time.perf_counter()
sim._check(sim.L.tp_get_state(sim.h, C.cast(h_out.data_ptr(), dp)))
t2 = time.perf_counter()
print(f"after steps: sync {1e3*(t1-t0):.2f} ms  get {1e3*(t2-t1):.1f} ms")
