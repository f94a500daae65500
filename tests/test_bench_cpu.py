"""Host logic of bench.py and the weak-scaling workload, no GPU needed."""
import numpy as np

import bench
from paper_2104_06784_b200 import scenarios


class _FakeSim:
    """Steps of fixed dt toward t_next with exact hits, like tp_steps (solver.cpp:637-649)."""

    class _Cfg:
        class scaling:
            @staticmethod
            def t_unit():
                return 1.0
        t_end = 10.0
        dt_out = 1.0

    def __init__(self, dt):
        self.cfg = self._Cfg()
        self.dt = dt
        self.calls = []

    def steps(self, t, t_next, k, t_end=None):
        self.calls.append((t, t_next, k))
        n, hit = 0, False
        while n < k and t < t_end:
            dt = min(self.dt, t_next - t)
            hit = dt == t_next - t
            t = t_next if hit else t + dt
            n += 1
            if hit:
                break
        return t, n, hit


def test_runclock_follows_output_schedule():
    sim = _FakeSim(0.3)
    clock = bench.RunClock(sim)
    assert clock.advance(7) == 7
    # 0.3, 0.6, 0.9, hit at 1.0 (next_out -> 2.0), 1.3, 1.6, 1.9
    assert abs(clock.t - 1.9) < 1e-12
    assert clock.next_out == 2.0
    assert sim.calls[0][1] == 1.0 and sim.calls[1][1] == 2.0
    # stops at t_end
    assert clock.advance(1000) < 1000 and clock.t == 10.0


def test_stacked_scenario_copies_rows():
    base = scenarios.c2_valley(40, 24)
    st = scenarios.stacked(base, 3)
    assert st.z.shape == (72, 40) and st.h0.shape == (72, 40)
    for k in range(3):
        np.testing.assert_array_equal(st.z[24 * k:24 * (k + 1)], base.z)
        np.testing.assert_array_equal(st.h0[24 * k:24 * (k + 1)], base.h0)


def test_reference_arm_runs_the_weak_scaling_grid():
    """--impl reference at --gpus N times the reference on the grid our arm runs at N
    (N row-stacked copies), rank 0 only; one JSON line with the reference keys."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "2",
                          "--warmup", "3", "--ncols", "96", "--nrows", "64"],
                         cwd=root, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-500:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["config"]["grid"] == [96, 128]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["value"] == d["value"]
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    quiet = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1"],
                           cwd=root, capture_output=True, text=True, timeout=600, env=env)
    assert quiet.returncode == 0 and not quiet.stdout.strip()


def test_balanced_decomposition_follows_wet_rows():
    """Strong scaling (bench.py --scaling strong): slab boundaries split the wet-tile work
    of the initial state evenly, not the rows."""
    from paper_2104_06784_b200.distributed import decompose_balanced, row_work
    sc = scenarios.c4_terrain(400, 300)
    w = row_work(sc)
    assert w.shape == (300,) and w.max() > 0
    for parts in (2, 3, 4, 8):
        p = decompose_balanced(w, parts)
        assert p[0][0] == 0 and p[-1][1] == 300
        assert all(a[1] == b[0] for a, b in zip(p[:-1], p[1:]))
        assert all(r1 - r0 >= 2 for r0, r1 in p)
        loads = [w[r0:r1].sum() + 0.05 * w.mean() * (r1 - r0) for r0, r1 in p]
        # each slab within one row's work of the mean (rows are indivisible)
        assert max(loads) - min(loads) <= 2 * (w.max() + 0.05 * w.mean()) + 1e-9, (parts, loads)
    # a release in the top quarter only: the top slabs get fewer rows
    sc2 = scenarios.c2_valley(160, 200)
    p = decompose_balanced(row_work(sc2), 4)
    sizes = [r1 - r0 for r0, r1 in p]
    assert sizes != [50, 50, 50, 50]
