import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.simulator import Simulator
sc = scenarios.c1_hill(32)
sim = Simulator.from_scenario(sc, fastdiv=bool(int(sys.argv[1]) if len(sys.argv) > 1 else 1))
sim.apply_boundaries(0.0)
dt = sim.compute_dt(0.0, 1e9)
print("dt", dt)
sim.advance_step(dt, 0.0)
print("ok", sim.state().sum())
