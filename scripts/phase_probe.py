"""Per-phase warp-cycle breakdown of the stage kernels (development probe).
usage: python scripts/phase_probe.py [scenario] [n] [steps]   (needs `make -C paper_2104_06784_b200/csrc timing`)"""
import ctypes as C, os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["TPFLOW_B200_LIB"] = os.path.join(HERE, "paper_2104_06784_b200", "libtpflow_b200_timing.so")
sys.path.insert(0, HERE)
from paper_2104_06784_b200 import scenarios, _lib
from paper_2104_06784_b200.simulator import Simulator
name = sys.argv[1] if len(sys.argv) > 1 else "wet"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
sc = scenarios.SCENARIOS[name](n, n) if name != "c1" else scenarios.c1_hill(n)
sim = Simulator.from_scenario(sc)
L = _lib.lib()
buf = (C.c_ulonglong * 38)()
sim.steps(0.0, 1e9, 8, t_end=1e9)
sim.synchronize()
L.tp_debug_phase_cycles(buf, 1)
sim.steps(0.0, 1e9, steps, t_end=1e9)
sim.synchronize()
L.tp_debug_phase_cycles(buf, 0)
names = ["loop top", "wait S/G TMA", "dry scan", "dry barrier", "phase1 work", "phase1 barrier",
         "wait cell TMA", "phase2 work", "phase2 barrier", "phase3 tail", "phase3 barrier",
         "p3 div+visc+upd", "p3 cap", "p3 heun", "p3 epilogue", "-"]
for st, label in ((0, "predictor"), (1, "corrector")):
    v = list(buf[19 * st: 19 * st + 19])
    tot = sum(v[:16])
    w = max(v[16], 1)
    print(f"{label}: warps {v[16]}  total {tot / w:.0f} cycles/warp; warp lifetime {v[17] / w:.0f} cycles, "
          f"{v[18] / w / 1e3:.1f} us (globaltimer)")
    for k in range(15):
        print(f"   {names[k]:16s} {100 * v[k] / tot:5.1f}%")
