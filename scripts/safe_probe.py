"""Active / safe tile counts over time (development probe).  usage: safe_probe.py cfg n steps"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.simulator import Simulator
name, n, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
sc = scenarios.SCENARIOS[name](n, n)
sim = Simulator.from_scenario(sc)
t = 0.0
for k in range(0, steps, 10):
    t, m, _ = sim.steps(t, 1e9, 10, t_end=1e9)
    p, c, tot = sim.active_tiles()
    print(f"step {k+10}: active {c}/{tot} safe {sim.safe_tiles()}")
