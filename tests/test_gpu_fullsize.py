"""Parity at BASELINE.json's full sizes (configs C2, C3, C4 and the C5 8192^2 point).

* C2 2048^2, C3 4096x2048 (Mode-II) and C4 6000x4000 run a bounded number of steps
  on the GPU and in the reference itself (oracle/_ref, BackendConfig::parallel with all
  host cores: its results are lane-count independent) from the same
  inputs; every dt and every padded state value must be bit-identical.
* C4 is also run for 20 steps, and row-split into 2 (equal rows) and 4 (equal work,
  decompose_balanced: the strong-scaling split of bench.py --scaling strong) peer-joined
  slabs on one GPU, bit-identical to the reference's single domain.
* 8192^2 (C5, the north-star grid): 5 steps bit for bit against the reference itself
  (~30 GB of host memory, ~3 s per step on 16 host cores), and size-independent
  properties over longer runs: (1) the mass balance of the reference's own audit
  (final = initial + injected - outflow + clipped, config.hpp:60-75) to round-off;
  (2) dry-tile skipping on/off gives bit-identical trajectories (the skip is exact by
  construction, DESIGN.md §3 item 5); (3) two row slabs joined by the device-resident
  peer exchange equal the single-domain run bit for bit.
"""
import os

import numpy as np
import pytest

from paper_2104_06784_b200 import scenarios
from tests.util import assert_bitwise

pytestmark = pytest.mark.gpu


def _lanes() -> int:
    return max(1, min(32, os.cpu_count() or 1))


def _pair(sc, kind):
    from oracle.oracle import OracleSim
    from paper_2104_06784_b200.simulator import Simulator
    return OracleSim(sc, kind, lanes=_lanes()), Simulator.from_scenario(sc)


def _run_intervals(ref, sim, t_end, interval, max_steps):
    """Both sides through the run loop's output schedule until max_steps steps."""
    t_r = t_g = 0.0
    done = 0
    k = 1
    while done < max_steps and t_r < t_end:
        t_next = min(k * interval, t_end)
        t_r, dts_r, hit_r = ref.steps(t_r, t_next, max_steps - done, t_end=t_end)
        t_g, dts_g, hit_g = sim.steps(t_g, t_next, max_steps - done, t_end=t_end, record_dts=True)
        assert_bitwise(np.asarray(dts_g), np.asarray(dts_r), f"dt sequence of interval {k}")
        assert t_r == t_g and bool(hit_r) == bool(hit_g)
        done += len(dts_r)
        if hit_r:
            k += 1
    return done


@pytest.mark.parametrize("name", ["c2", "c3", "c4"])
def test_fullsize_bitwise_vs_reference(gpu, oracle_kind, name):
    if oracle_kind != "ref":
        pytest.skip("full-size parity runs against the compiled reference (oracle/_ref)")
    if name == "c2":
        sc, nsteps = scenarios.c2_valley(2048, 2048), 40
    elif name == "c3":
        sc, nsteps = scenarios.c3_channel(4096, 2048), 40
    else:
        sc, nsteps = scenarios.c4_terrain(6000, 4000), 20
    ref, sim = _pair(sc, "ref")
    tu = sc.config.scaling.t_unit()
    done = _run_intervals(ref, sim, sc.config.t_end / tu, sc.config.dt_out / tu, nsteps)
    assert done == nsteps
    assert_bitwise(sim.state(), ref.state(), f"{name} full-size state after {nsteps} steps")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


def test_c4_peer_slabs_bitwise_vs_reference(gpu, oracle_kind):
    """C4 6000x4000 (BASELINE configs[3], the Hsiaolin-scale terrain) row-split into 2 slabs
    of equal rows and 4 slabs of equal work (the strong-scaling decomposition), each set
    joined by the device-resident peer exchange (tp_peer.cu) and time-sliced on one GPU:
    dt and the interior after 8 steps bit-identical to the reference's single domain."""
    if oracle_kind != "ref":
        pytest.skip("full-size parity runs against the compiled reference (oracle/_ref)")
    import torch
    from oracle.oracle import OracleSim
    from paper_2104_06784_b200.distributed import (CudaSlab, PeerGroup, assemble, decompose,
                                                   decompose_balanced, row_work)
    sc = scenarios.c4_terrain(6000, 4000)
    ref = OracleSim(sc, "ref", lanes=_lanes())
    t_r, d_r, _ = ref.steps(0.0, 1.0e9, 8, t_end=1.0e9)
    want = ref.state()[:, 3:-3, 3:-3]
    del ref
    for parts in (decompose(sc.nrows, 2), decompose_balanced(row_work(sc), 4)):
        slabs = [CudaSlab(sc, r, stream=torch.cuda.Stream()) for r in parts]
        t_g, n_g, _ = PeerGroup(slabs).steps(0.0, 1.0e9, 8, t_end=1.0e9)
        assert n_g == len(d_r) == 8 and t_g == t_r
        assert_bitwise(assemble([s.state() for s in slabs]), want, f"C4 interior, slabs {parts}")
        for s in slabs:
            s.sim.close()
        torch.cuda.synchronize()


@pytest.fixture(scope="module")
def c5():
    return scenarios.c2_valley(8192, 8192)


def _drift(a, ms, mf):
    """config.hpp:60-75 MassAudit::drift per phase, relative to initial + injected."""
    out = []
    for p, m in ((0, ms), (1, mf)):
        initial, injected, outflow, clipped = a[5 * p], a[5 * p + 2], a[5 * p + 3], a[5 * p + 4]
        out.append(abs(m - (initial + injected - outflow + clipped)) / max(abs(initial) + injected, 1e-300))
    return out


def test_c5_8192_mass_balance(gpu, c5):
    from paper_2104_06784_b200.simulator import Simulator
    sim = Simulator.from_scenario(c5)
    sim.reset_audit()
    ms0, mf0 = sim.interior_mass_device()
    a = sim.audit_array()
    a[0], a[5] = ms0, mf0
    sim._set_audit(a)
    t, dts, _ = sim.steps(0.0, 1.0e9, 40, t_end=1.0e9, record_dts=True)
    assert len(dts) == 40 and t > 0.0
    ms, mf = sim.interior_mass_device()
    for d in _drift(sim.audit_array(), ms, mf):
        assert d < 1e-12, d
    s = sim.state()
    assert np.isfinite(s).all()
    assert (s[0:2] >= 0.0).all()


def test_c5_8192_skip_equals_full_list(gpu, c5):
    from paper_2104_06784_b200.simulator import Simulator
    a = Simulator.from_scenario(c5)
    t_a, d_a, _ = a.steps(0.0, 1.0e9, 10, t_end=1.0e9, record_dts=True)
    s_a = a.state()
    a.close()
    b = Simulator.from_scenario(c5)
    b.set_option("skip_dry", 0)
    t_b, d_b, _ = b.steps(0.0, 1.0e9, 10, t_end=1.0e9, record_dts=True)
    assert t_a == t_b
    assert_bitwise(np.asarray(d_b), np.asarray(d_a), "dt sequence")
    assert_bitwise(b.state(), s_a, "8192^2 state, skip on vs off")


def test_c5_8192_peer_slabs_equal_single(gpu, c5):
    import torch
    from paper_2104_06784_b200.distributed import CudaSlab, PeerGroup, assemble, decompose
    from paper_2104_06784_b200.simulator import Simulator
    one = Simulator.from_scenario(c5)
    t1, d1, _ = one.steps(0.0, 1.0e9, 6, t_end=1.0e9, record_dts=True)
    s1 = one.state()[:, 3:-3, 3:-3]
    one.close()
    slabs = [CudaSlab(c5, r, stream=torch.cuda.Stream()) for r in decompose(c5.nrows, 2)]
    t2, n2, _ = PeerGroup(slabs).steps(0.0, 1.0e9, 6, t_end=1.0e9)
    assert t1 == t2 and n2 == len(d1)
    assert_bitwise(assemble([s.state() for s in slabs]), s1, "8192^2 interior, 2 peer slabs vs one domain")


def test_c5_8192_bitwise_vs_reference(gpu, oracle_kind, c5):
    """The north-star grid (8192^2 C2-style valley) for 5 steps against the reference itself
    (oracle/_ref, BackendConfig::parallel on all host cores): every dt and every padded
    state value bit-identical (solver.cpp:496-580, :637-649)."""
    if oracle_kind != "ref":
        pytest.skip("full-size parity runs against the compiled reference (oracle/_ref)")
    from oracle.oracle import OracleSim
    from paper_2104_06784_b200.simulator import Simulator
    sim = Simulator.from_scenario(c5)
    t_g, d_g, _ = sim.steps(0.0, 1.0e9, 5, t_end=1.0e9, record_dts=True)
    got = sim.state()
    sim.close()
    ref = OracleSim(c5, "ref", lanes=_lanes())
    t_r, d_r, _ = ref.steps(0.0, 1.0e9, 5, t_end=1.0e9)
    assert len(d_r) == 5 and t_g == t_r
    assert_bitwise(np.asarray(d_g), np.asarray(d_r), "8192^2 dt sequence")
    assert_bitwise(got, ref.state(), "8192^2 state after 5 steps")
