"""Per-phase warp-cycle breakdown of the stage kernels along a scenario's run schedule
(development probe; needs `make -C paper_2104_06784_b200/csrc timing`).
usage: python scripts/phase_probe_run.py config ncols nrows steps [wide_tiles]"""
import ctypes as C, os, sys
HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ["TPFLOW_B200_LIB"] = os.path.join(HERE, "paper_2104_06784_b200", "libtpflow_b200_timing.so")
sys.path.insert(0, HERE)
import bench
from paper_2104_06784_b200 import _lib
from paper_2104_06784_b200.simulator import Simulator
cfg, nc, nr, steps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
sc = bench.scenario_for(cfg, nc, nr)
sim = Simulator.from_scenario(sc)
if len(sys.argv) > 5:
    sim.set_option("wide_tiles", int(sys.argv[5]))
clock = bench.RunClock(sim)
L = _lib.lib()
buf = (C.c_ulonglong * 38)()
clock.advance(20)
sim.synchronize()
L.tp_debug_phase_cycles(buf, 1)
clock.advance(steps)
sim.synchronize()
L.tp_debug_phase_cycles(buf, 0)
names = ["loop top", "wait S/G TMA", "-", "-", "phase1 work", "phase1 barrier",
         "wait cell TMA", "phase2 work", "phase2 barrier", "phase3 tail", "phase3 barrier",
         "p3 div+visc+upd", "p3 cap", "p3 heun", "p3 epilogue", "-"]
print(f"{cfg} {nc}x{nr}, {steps} steps, active tiles {sim.active_tiles()}")
for st, label in ((0, "predictor"), (1, "corrector")):
    v = list(buf[19 * st: 19 * st + 19])
    tot = sum(v[:16])
    w = max(v[16], 1)
    print(f"{label}: warps {v[16]}  total {tot / w:.0f} cycles/warp; warp lifetime {v[17] / w:.0f} cycles, "
          f"{v[18] / w / 1e3:.2f} us (globaltimer)")
    for k in range(15):
        if names[k] != "-":
            print(f"   {names[k]:16s} {100 * v[k] / max(tot, 1):5.1f}%  {v[k] / w:8.0f} cyc/warp")
