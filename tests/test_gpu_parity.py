"""CUDA path vs the CPU reference on identical inputs (the parity gate).

Bit-exact: with --fmad=false, IEEE div/sqrt, host-hoisted pow/tan and the
reference's expression trees, the sm_100a kernels reproduce the reference
Simulator bit for bit: every dt, every padded state value (ghosts included).
The north_star tolerance (relative L1/Linf <= 1e-9, identical dt) is therefore
met with margin; tests assert the stronger bitwise property.
"""
import numpy as np
import pytest

from paper_2104_06784_b200 import scenarios
from paper_2104_06784_b200.config import NumericsError
from tests.util import assert_bitwise, rel_err

pytestmark = pytest.mark.gpu


def _pair(sc, kind, fastdiv=True, wide=None):
    """wide: None = automatic (wide stage CTAs while the lists are shorter than the SM count,
    i.e. almost always on these small grids), True / False = forced."""
    from oracle.oracle import OracleSim
    from paper_2104_06784_b200.simulator import Simulator
    sim = Simulator.from_scenario(sc, fastdiv=fastdiv)
    if wide is not None:
        sim.set_option("wide_tiles", 1 << 30 if wide else 0)
    return OracleSim(sc, kind), sim


def test_division_identity(gpu):
    import ctypes as C
    bad = C.c_ulonglong()
    assert gpu.tp_selftest_division(0, 50_000_000, 2104, C.byref(bad)) == 0
    assert bad.value == 0


def _minmod_reference(a, b):
    """solver.hpp:17-21 element-wise: a>0&&b>0 -> std::min, a<0&&b<0 -> std::max, else 0.0."""
    out = np.zeros_like(a)
    pos = (a > 0.0) & (b > 0.0)
    neg = (a < 0.0) & (b < 0.0)
    out[pos] = np.where(b < a, b, a)[pos]   # std::min(a, b) = (b < a) ? b : a
    out[neg] = np.where(a < b, b, a)[neg]   # std::max(a, b) = (a < b) ? b : a
    return out


def test_minmod_bitwise(gpu):
    """Device limited_slope vs the reference on random, tied, signed-zero, subnormal and
    infinite operands (a nvcc contraction once turned `M < 0 ? M : 0` into -0.0)."""
    import ctypes as C
    rng = np.random.default_rng(2104)
    n = 1 << 21
    bits = rng.integers(0, 2**63, size=(2, n), dtype=np.int64).view(np.uint64)
    bits ^= rng.integers(0, 2, size=(2, n), dtype=np.uint64) << np.uint64(63)
    ab = bits.view(np.float64).copy()
    ab[~np.isfinite(ab)] = 1.0
    special = np.array([0.0, -0.0, 1.0, -1.0, 5e-324, -5e-324, 2.0**-1022, np.inf, -np.inf, 3.0, -3.0])
    k = n // 4
    ab[0, :k] = special[rng.integers(0, len(special), k)]
    ab[1, k:2 * k] = special[rng.integers(0, len(special), k)]
    ab[1, 2 * k:3 * k] = ab[0, 2 * k:3 * k] * rng.choice([1.0, 0.5, -1.0, 2.0], k)
    a, b = np.ascontiguousarray(ab[0]), np.ascontiguousarray(ab[1])
    out = np.empty(n)
    dp = C.POINTER(C.c_double)
    assert gpu.tp_selftest_minmod(0, n, a.ctypes.data_as(dp), b.ctypes.data_as(dp), out.ctypes.data_as(dp)) == 0
    ref = _minmod_reference(a, b)
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("fastdiv", [False, True])
def test_step_api_bitwise_c1(gpu, oracle_kind, fastdiv):
    """apply_boundaries / compute_dt / advance_step one by one (solver.hpp:41-47)."""
    sc = scenarios.c1_hill(48)
    ref, sim = _pair(sc, oracle_kind, fastdiv)
    assert_bitwise(sim.state(), ref.state(), "initial state")
    t, t_next = 0.0, 1.0e9
    for n in range(12):
        ref.apply_boundaries(t)
        sim.apply_boundaries(t)
        assert_bitwise(sim.state(), ref.state(), f"after apply_boundaries, step {n}")
        dr = ref.compute_dt(t, t_next)
        dg = sim.compute_dt(t, t_next)
        assert dg == dr, (n, dg, dr)
        ref.advance_step(dr, t)
        sim.advance_step(dr, t)
        assert_bitwise(sim.state(), ref.state(), f"after advance_step, step {n}")
        t += dr
    a_r, a_g = ref.audit(), sim.audit_array()
    np.testing.assert_allclose(a_g, a_r, rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("wide", [False, True])
@pytest.mark.parametrize("fastdiv", [False, True])
def test_trajectory_c1_device_loop(gpu, oracle_kind, fastdiv, wide):
    """tp_steps (device-resident loop, CUDA graphs) == the reference run loop, 150 steps,
    with the production stage CTAs and with the wide (one tile per SM) ones."""
    sc = scenarios.c1_hill(96)
    ref, sim = _pair(sc, oracle_kind, fastdiv, wide)
    tr, dts_r, hr = ref.steps(0.0, 1.0e9, 150, t_end=1.0e9)
    tg, dts_g, hg = sim.steps(0.0, 1.0e9, 150, t_end=1.0e9, record_dts=True)
    assert len(dts_g) == len(dts_r) == 150
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert tg == tr and hg == hr
    assert_bitwise(sim.state(), ref.state(), "state after 150 steps")
    l1, linf = rel_err(sim.state(), ref.state())
    assert l1 <= 1e-9 and linf <= 1e-9


def test_trajectory_output_hits(gpu, oracle_kind):
    """exact-hit truncation at output times (solver.cpp:638-648)."""
    sc = scenarios.c1_hill(64)
    ref, sim = _pair(sc, oracle_kind)
    t_r = t_g = 0.0
    for k in range(1, 4):
        t_next = 2.5 * k
        t_r, dts_r, h_r = ref.steps(t_r, t_next, 10_000, t_end=1e9)
        t_g, dts_g, h_g = sim.steps(t_g, t_next, 10_000, t_end=1e9, record_dts=True)
        assert h_r and h_g and t_r == t_g == t_next
        assert_bitwise(dts_g, dts_r, f"dts to output {k}")
    assert_bitwise(sim.state(), ref.state(), "state at output times")


@pytest.mark.parametrize("opts", [{"merge_post": 0}, {"graph_steps": 1}, {"graph_steps": 3},
                                  {"graph_steps": 64}, {"merge_post": 0, "graph_steps": 5}])
def test_loop_structure_options_bitwise(gpu, oracle_kind, opts):
    """The device loop's structure is not semantics: post merged into the next pre or not
    (prepost_kernel), and replay batches of any length (power-of-two graphs sized to the next
    output), give the reference's dt sequence and state bit for bit along an output schedule
    with hits, a Mode-II inflow and a run past the hydrograph."""
    sc = scenarios.four_side_inflow(48, 40)
    ref, sim = _pair(sc, oracle_kind)
    for k, v in opts.items():
        sim.set_option(k, v)
    tu = sc.config.scaling.t_unit()
    t_r = t_g = 0.0
    t_end = sc.config.t_end / tu
    for k in range(1, 41):
        t_next = min(k * sc.config.dt_out / tu, t_end)
        t_r, dts_r, _ = ref.steps(t_r, t_next, 100_000, t_end=t_end)
        t_g, dts_g, _ = sim.steps(t_g, t_next, 100_000, t_end=t_end, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dts interval {k} {opts}")
        assert t_r == t_g
        if opts.get("merge_post", 1) == 0:  # five launches per step (and per no-op step)
            assert sim.kernel_launches() >= 5 * len(dts_g)
    assert_bitwise(sim.state(), ref.state(), f"state {opts}")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("wide", [False, True])
def test_mode2_channel_inflow(gpu, oracle_kind, wide):
    """Mode-II hydrograph inflow (solver.cpp:108-136, hydrograph.hpp:31-45)."""
    sc = scenarios.c3_channel(96, 48, t_end=30.0, dt_out=0.5)
    ref, sim = _pair(sc, oracle_kind, wide=wide)
    tu = sc.config.scaling.t_unit()
    t_r = t_g = 0.0
    for k in range(1, 9):
        t_next = min(k * 0.5 / tu, 30.0 / tu)
        t_r, dts_r, _ = ref.steps(t_r, t_next, 100_000, t_end=30.0 / tu)
        t_g, dts_g, _ = sim.steps(t_g, t_next, 100_000, t_end=30.0 / tu, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dts interval {k}")
        assert t_r == t_g
    assert_bitwise(sim.state(), ref.state(), "Mode-II state")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("t_end,dt_out", [(4.0, 1.0), (2.0, 0.7)])
def test_run_report_matches(gpu, oracle_kind, t_end, dt_out):
    """Simulator::run end to end: steps, snapshot times (incl. a last output at t_end that is
    not a multiple of dt_out), audit (solver.cpp:619-659)."""
    sc = scenarios.c1_hill(48, t_end=t_end, dt_out=dt_out)
    ref, sim = _pair(sc, oracle_kind)
    rep_r, snaps_r = ref.run()
    times = []
    rep_g = sim.run(sink=lambda s: times.append(s.t))
    assert rep_g.steps == int(rep_r[0])
    np.testing.assert_array_equal(np.array(times), snaps_r)
    a_g = np.array([rep_g.solid.initial, rep_g.solid.final_mass, rep_g.solid.injected, rep_g.solid.outflow,
                    rep_g.solid.clipped, rep_g.fluid.initial, rep_g.fluid.final_mass, rep_g.fluid.injected,
                    rep_g.fluid.outflow, rep_g.fluid.clipped])
    np.testing.assert_array_equal(a_g[[0, 1, 5, 6]], rep_r[2:][[0, 1, 5, 6]])  # Kahan masses: exact
    np.testing.assert_allclose(a_g, rep_r[2:], rtol=1e-12, atol=1e-300)
    assert_bitwise(sim.state(), ref.state(), "state after run")


@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(64), lambda: scenarios.c4_terrain(120, 90),
                                  lambda: scenarios.c3_channel(96, 48)])
def test_device_geometry_bitwise(gpu, oracle_kind, make):
    """Geometry built on the device (tp_geometry.cu) vs the reference's compute_geometry on
    the extended DEM (terrain.cpp:113-215), all 14 fields, whole grid and a middle slab."""
    from paper_2104_06784_b200.simulator import Simulator
    from oracle.oracle import OracleSim
    sc = make()
    ref = OracleSim(sc, oracle_kind).geometry()
    sim = Simulator.from_scenario(sc, init=False)
    assert_bitwise(sim.geometry(), ref, "device geometry")
    r0, r1 = sc.nrows // 3, 2 * sc.nrows // 3
    slab = Simulator.from_scenario(sc, rows=(r0, r1), init=False)
    assert_bitwise(slab.geometry(), ref[:, r0:r1 + 6, :], "device geometry of a slab")


def test_device_mass(gpu, oracle_kind):
    """Device interior-mass reduction vs the reference's serial KahanSum (solver.cpp:582-588)."""
    sc = scenarios.wet_valley(200, 170)
    ref, sim = _pair(sc, oracle_kind)
    ref.steps(0.0, 1.0e9, 10, t_end=1.0e9)
    sim.steps(0.0, 1.0e9, 10, t_end=1.0e9)
    ms_r, mf_r = ref.interior_mass()
    ms_h, mf_h = sim.interior_mass()
    ms_d, mf_d = sim.interior_mass_device()
    assert (ms_h, mf_h) == (ms_r, mf_r)  # host path: the reference's Kahan bit for bit
    assert abs(ms_d - ms_r) <= 4e-16 * abs(ms_r) and abs(mf_d - mf_r) <= 4e-16 * abs(mf_r)


@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(64), lambda: scenarios.wet_valley(80, 72)])
def test_snapshot_bitwise(gpu, oracle_kind, make):
    """Simulator::snapshot (solver.cpp:590-617) computed on the device, field by field."""
    sc = make()
    ref, sim = _pair(sc, oracle_kind)
    tr, _, _ = ref.steps(0.0, 1.0e9, 25, t_end=1.0e9)
    tg, _, _ = sim.steps(0.0, 1.0e9, 25, t_end=1.0e9)
    assert tr == tg
    snap_r = ref.snapshot(tr)
    snap_g = sim.snapshot(tg)
    got = np.stack([snap_g.h_total, snap_g.phi_s, snap_g.vX_s, snap_g.vY_s, snap_g.vX_f, snap_g.vY_f])
    assert_bitwise(got, snap_r.reshape(got.shape), "snapshot fields")


def test_negative_thickness_error_matches(gpu, oracle_kind):
    """regularize's NumericsError text (solver.cpp:147-152)."""
    sc = scenarios.c1_hill(32)
    ref, sim = _pair(sc, oracle_kind)
    s = ref.state()
    s[0, 10, 12] = -1e-6
    s[1, 10, 15] = -2e-6
    ref.set_state(s)
    sim.set_state(s)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError) as er:
        ref.regularize()
    with pytest.raises(NumericsError) as eg:
        sim.regularize()
    assert str(eg.value) == str(er.value)


@pytest.mark.parametrize("wide", [False, True])
@pytest.mark.parametrize("name", ["c2", "wet", "c4"])
def test_trajectory_other_terrains(gpu, oracle_kind, name, wide):
    """valley (mostly dry: exercises the dry-tile fast path), fully wet valley, seeded terrain."""
    sc = {"c2": lambda: scenarios.c2_valley(160, 144), "wet": lambda: scenarios.wet_valley(128, 112),
          "c4": lambda: scenarios.c4_terrain(120, 90)}[name]()
    ref, sim = _pair(sc, oracle_kind, wide=wide)
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 60, t_end=1.0e9)
    tg, dts_g, _ = sim.steps(0.0, 1.0e9, 60, t_end=1.0e9, record_dts=True)
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert tg == tr
    assert_bitwise(sim.state(), ref.state(), f"{name} state after 60 steps")


def test_signed_zero_state(gpu, oracle_kind):
    """-0.0 entries in dry cells must not take the all-(+0.0) dry-tile shortcut."""
    sc = scenarios.c1_hill(64)
    ref, sim = _pair(sc, oracle_kind)
    s = ref.state()
    s[2:, 3:20, 3:20] = -0.0
    s[0, 5, 5] = -0.0
    ref.set_state(s)
    sim.set_state(s)
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 20, t_end=1.0e9)
    tg, dts_g, _ = sim.steps(0.0, 1.0e9, 20, t_end=1.0e9, record_dts=True)
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert_bitwise(sim.state(), ref.state(), "state with signed zeros")


def test_signed_zero_thickness_in_wet_region(gpu, oracle_kind):
    """-0.0 thickness cells beside wet ones (allowed in safe tiles): the safe-tile face code
    relies on every minmod edge of a non-negative thickness field being +0 or positive."""
    sc = scenarios.wet_valley(64, 60)
    ref, sim = _pair(sc, oracle_kind)
    s = ref.state()
    s[0:2, 20:24, 10:50] = -0.0
    s[2:, 20:24, 10:50] = -0.0
    s[1, 40:42, 30:33] = -0.0
    ref.set_state(s)
    sim.set_state(s)
    for k in range(3):
        tr, dts_r, _ = ref.steps(0.0 if k == 0 else tr, 1.0e9, 15, t_end=1.0e9)
        tg, dts_g, _ = sim.steps(0.0 if k == 0 else tg, 1.0e9, 15, t_end=1.0e9, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dt sequence {k}")
        assert_bitwise(sim.state(), ref.state(), f"state after leg {k}")
    assert sim.safe_tiles() > 0


def test_safe_window_edges(gpu, oracle_kind):
    """Values outside the safe-tile window (nonzero magnitudes below 2^-200 or
    at/above 2^200, subnormals) mark their tile and its neighbours unsafe, which then take
    the checked FASTDIV path; the rest of the grid keeps the safe path.  Both must match."""
    sc = scenarios.wet_valley(96, 80)
    ref, sim = _pair(sc, oracle_kind)
    ref.steps(0.0, 1.0e9, 5, t_end=1.0e9)  # a developed state with nonzero momenta
    s = ref.state()
    s[0, 10, 10] = 2.0 ** -201          # just below the window (thickness)
    s[3, 30, 40] = 5e-310               # subnormal momentum
    s[4, 50, 20] = -(2.0 ** -200)       # the window's lower edge: still safe
    s[2, 60, 70] = 2.0 ** -180          # inside window A, outside window B
    s[1, 40, 60] = 2.0 ** -101          # just outside window B
    s[3, 20, 80] = -(2.0 ** 99)         # inside window B
    s[5, 70, 90] = 2.0 ** 200           # the window's upper edge: unsafe
    ref.set_state(s)
    sim.set_state(s)
    # two stages warm the flags (set_state marks every tile unknown), then steps run
    # with a mix of safe and unsafe tiles
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 30, t_end=1.0e9)
    t1, dts_1, _ = sim.steps(0.0, 1.0e9, 2, t_end=1.0e9, record_dts=True)
    act_p, act_c, ntiles = sim.active_tiles()
    safe = sim.safe_tiles()
    assert 0 < safe < act_c, (safe, act_c)  # both paths ran in the last corrector
    tg, dts_g, _ = sim.steps(t1, 1.0e9, 28, t_end=1.0e9, record_dts=True)
    assert_bitwise(np.concatenate([dts_1, dts_g]), dts_r, "dt sequence")
    assert_bitwise(sim.state(), ref.state(), "state around out-of-window values")


def test_set_state_exact_flags(gpu, oracle_kind):
    """tp_set_state scans the new state's tile flags (flag_scan_kernel) instead of marking
    every tile unknown: a state round-tripped through the host lists exactly the tiles the
    uninterrupted run lists, and both runs stay bit-identical to the reference (dt, state)."""
    from paper_2104_06784_b200.simulator import Simulator
    sc = scenarios.c1_hill(160)
    ref, sim = _pair(sc, oracle_kind)
    other = Simulator.from_scenario(sc)
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 40, t_end=1.0e9)
    t1, _, _ = sim.steps(0.0, 1.0e9, 20, t_end=1.0e9)
    t2, _, _ = other.steps(0.0, 1.0e9, 20, t_end=1.0e9)
    other.set_state(other.state())  # host round trip: flags and lambda rebuilt from the state
    t1, d1, _ = sim.steps(t1, 1.0e9, 1, t_end=1.0e9, record_dts=True)
    t2, d2, _ = other.steps(t2, 1.0e9, 1, t_end=1.0e9, record_dts=True)
    assert sim.active_tiles() == other.active_tiles()
    assert_bitwise(d2, d1, "dt after the round trip")
    sim.steps(t1, 1.0e9, 19, t_end=1.0e9)
    other.steps(t2, 1.0e9, 19, t_end=1.0e9)
    assert_bitwise(other.state(), ref.state(), "state after set_state")
    assert_bitwise(sim.state(), ref.state(), "state")


@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(96), lambda: scenarios.wet_valley(96, 80),
                                  lambda: scenarios.c3_channel(96, 48, t_end=30.0, dt_out=0.5)])
def test_full_tile_list_bitwise(gpu, oracle_kind, make):
    """option skip_dry=0 (every tile listed, no dry-tile skipping) is bit-identical too."""
    sc = make()
    ref, sim = _pair(sc, oracle_kind)
    sim.set_option("skip_dry", 0)
    t_next = 0.5 / sc.config.scaling.t_unit() if sc.config.inflow else 1e9
    tr, dts_r, _ = ref.steps(0.0, t_next, 80, t_end=1e9)
    tg, dts_g, _ = sim.steps(0.0, t_next, 80, t_end=1e9, record_dts=True)
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert_bitwise(sim.state(), ref.state(), "full-list state")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("seed", list(range(1, 9)))
def test_random_api_sequences(gpu, oracle_kind, seed):
    """Random interleavings of the public API (device loop, step pieces, regularize,
    state uploads that wet, dry out, zero or shrink regions) stay bit-identical to the
    reference: exercises the tile flags, the dry-tile lists and the safe-tile window
    across every path that writes a state buffer."""
    rng = np.random.default_rng(seed)
    sc = scenarios.wet_valley(72, 60) if seed % 2 else scenarios.c1_hill(64)
    ref, sim = _pair(sc, oracle_kind)
    t = 0.0
    for _ in range(12):
        op = rng.choice(["loop", "pieces", "perturb", "regularize"])
        if op == "loop":
            k = int(rng.integers(1, 15))
            t_r, _, _ = ref.steps(t, 1.0e9, k, t_end=1.0e9)
            t_g, _, _ = sim.steps(t, 1.0e9, k, t_end=1.0e9)
            assert t_r == t_g
            t = t_r
        elif op == "pieces":
            ref.apply_boundaries(t)
            sim.apply_boundaries(t)
            dt_r, dt_g = ref.compute_dt(t, 1.0e9), sim.compute_dt(t, 1.0e9)
            assert dt_r == dt_g
            ref.advance_step(dt_r, t)
            sim.advance_step(dt_g, t)
            t = t + dt_r
        elif op == "perturb":
            s = ref.state()
            j0, i0 = int(rng.integers(3, s.shape[1] - 20)), int(rng.integers(3, s.shape[2] - 20))
            blk = (slice(None), slice(j0, j0 + 17), slice(i0, i0 + 17))
            kind = rng.integers(0, 4)
            if kind == 0:
                s[blk] = 0.0                                        # dry out a block
            elif kind == 1:
                s[0:2][:, blk[1], blk[2]] += rng.uniform(0.0, 0.3, (2, 17, 17))  # wet it
            elif kind == 2:
                s[blk] *= 2.0 ** -110                               # below the safe window
            else:
                s[2:][:, blk[1], blk[2]] = -s[2:][:, blk[1], blk[2]]  # reverse the flow
            ref.set_state(s)
            sim.set_state(s)
        else:
            ref.regularize()
            sim.regularize()
        assert_bitwise(sim.state(), ref.state(), f"state after {op}")


@pytest.mark.parametrize("shape", [(2, 2), (3, 5), (5, 3), (16, 15), (17, 16), (15, 14), (33, 31), (1 + 16 * 3, 2)])
def test_small_and_ragged_grids(gpu, oracle_kind, shape):
    """Grids smaller than one 16x15 tile, exactly one tile, one cell more or less, and a
    2-row strip: partial tiles, clipped TMA boxes and ring-only tile lists."""
    ncols, nrows = shape
    sc = scenarios.wet_valley(ncols, nrows)
    ref, sim = _pair(sc, oracle_kind)
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 25, t_end=1.0e9)
    tg, dts_g, _ = sim.steps(0.0, 1.0e9, 25, t_end=1.0e9, record_dts=True)
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert_bitwise(sim.state(), ref.state(), f"state {ncols}x{nrows}")


def test_config0_c1_1000_steps(gpu, oracle_kind):
    """BASELINE configs[0] end to end: the 256^2 hill release for 1000 steps, every dt and
    the final state bit-identical to the reference (plus the north-star 1e-9 gate)."""
    sc = scenarios.c1_hill(256)
    ref, sim = _pair(sc, oracle_kind)
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 1000, t_end=1.0e9)
    tg, dts_g, _ = sim.steps(0.0, 1.0e9, 1000, t_end=1.0e9, record_dts=True)
    assert len(dts_r) == 1000
    assert_bitwise(dts_g, dts_r, "1000 dts")
    assert tg == tr
    g, r = sim.state(), ref.state()
    assert_bitwise(g, r, "state after 1000 steps")
    for f in range(6):
        l1, linf = rel_err(g[f], r[f])
        assert l1 <= 1e-9 and linf <= 1e-9
    ms_r, mf_r = ref.interior_mass()
    ms_g, mf_g = sim.interior_mass()
    assert (ms_g, mf_g) == (ms_r, mf_r)


@pytest.mark.parametrize("case", ["negative", "nonfinite"])
def test_step_errors_match(gpu, oracle_kind, case):
    """NumericsError raised inside a step (regularize after the predictor/corrector,
    solver.cpp:147-152; check_finite, :482-494): same message as the reference, through
    the device loop and through the step API."""
    from oracle.oracle import OracleError
    sc = scenarios.c1_hill(48)
    for api in ("loop", "pieces"):
        ref, sim = _pair(sc, oracle_kind)
        s = ref.state()
        if case == "negative":
            # negative thickness in a dry corner: it survives the predictor and its regularize throws
            s[0, 8, 9] = -1e-6
            s[1, 40, 10] = -3e-6
        else:
            # non-finite values inside the release (regularize would zero momenta of dry cells)
            s[0, 27, 37] = np.inf
            s[2, 26, 36] = np.nan
        ref.set_state(s)
        sim.set_state(s)
        with pytest.raises(OracleError) as er:
            if api == "loop":
                ref.steps(0.0, 1.0e9, 5, t_end=1.0e9)
            else:
                ref.apply_boundaries(0.0)
                ref.advance_step(ref.compute_dt(0.0, 1.0e9), 0.0)
        with pytest.raises(NumericsError) as eg:
            if api == "loop":
                sim.steps(0.0, 1.0e9, 5, t_end=1.0e9)
            else:
                sim.apply_boundaries(0.0)
                sim.advance_step(sim.compute_dt(0.0, 1.0e9), 0.0)
        assert str(eg.value) == str(er.value), api


@pytest.mark.parametrize("seed", list(range(8)))
def test_random_parameters_bitwise(gpu, oracle_kind, seed):
    """Non-default model parameters, scaling (ε = H/L ≠ 1, χ ≠ 1), CFL, h_dry and eps_h:
    every host-hoisted constant (tan δb, ε^χ, 1−α, ε·N_R, ...) and the safe-tile constant
    window must reproduce the reference's per-cell evaluation bit for bit."""
    rng = np.random.default_rng(700 + seed)
    kind = seed % 3
    if kind == 0:
        sc = scenarios.c4_terrain(56, 44, seed=2104 + seed)
    elif kind == 1:
        sc = scenarios.wet_valley(50, 46)
    else:
        sc = scenarios.c3_channel(64, 40, t_end=30.0, dt_out=0.5)
    p, s, cfg = sc.config.params, sc.config.scaling, sc.config
    p.delta_b = float(rng.uniform(5.0, 35.0))
    p.C_d = float(rng.uniform(0.0, 10.0))
    p.N_R = float(rng.uniform(20.0, 800.0))
    p.theta_b = float(rng.uniform(0.0, 10.0))
    p.phi_s0 = float(rng.uniform(0.2, 0.8))
    p.alpha_rho = float(rng.uniform(0.2, 1.0))
    p.chi = float(rng.choice([0.5, 1.0, 1.5, 2.0]))
    s.L = float(rng.choice([1.0, 2.0, 10.0]))
    s.H = float(rng.choice([0.5, 1.0, 4.0]))
    cfg.cfl = float(rng.uniform(0.05, 0.125))
    cfg.h_dry = float(10.0 ** rng.uniform(-12, -7))
    cfg.eps_h = float(10.0 ** rng.uniform(-8, -4))
    cfg.validate()
    ref, sim = _pair(sc, oracle_kind)
    assert_bitwise(sim.state(), ref.state(), "initial state")
    tu = s.t_unit()
    t_r = t_g = 0.0
    for k in range(1, 4):
        t_next = k * cfg.dt_out / tu if cfg.inflow else 1e9
        t_r, dts_r, _ = ref.steps(t_r, t_next, 20, t_end=cfg.t_end / tu)
        t_g, dts_g, _ = sim.steps(t_g, t_next, 20, t_end=cfg.t_end / tu, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dt sequence, leg {k}")
        assert t_r == t_g
    assert_bitwise(sim.state(), ref.state(), "state")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("shape", [(64, 48), (37, 29)])
def test_initial_velocity_bitwise(gpu, oracle_kind, shape):
    """set_initial_velocity (solver.cpp:57-81, init_velocity_kernel on the device): the
    initial momenta and 40 steps from a moving release are bit-identical."""
    sc = scenarios.moving_release(*shape)
    ref, sim = _pair(sc, oracle_kind)
    assert_bitwise(sim.state(), ref.state(), "initial state with velocity")
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 40, t_end=1.0e9)
    tg, dts_g, _ = sim.steps(0.0, 1.0e9, 40, t_end=1.0e9, record_dts=True)
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert tg == tr
    assert_bitwise(sim.state(), ref.state(), "state after 40 steps")


@pytest.mark.parametrize("shape", [(48, 40), (49, 46)])
def test_four_side_inflow_bitwise(gpu, oracle_kind, shape):
    """Mode-II inflow on W, N, S and E boundary cells (the SE corner cell on two sides),
    through and past the end of the hydrograph: dt, state and audit bit-identical.  49x46
    leaves a last tile of one column and one row, so the inner neighbour tiles' boxes reach
    the E / N inflow ghosts (listed through the per-tile inflow mask, never skipped)."""
    sc = scenarios.four_side_inflow(*shape)
    sc.hydrograph.validate(sc.ncols, sc.nrows)
    ref, sim = _pair(sc, oracle_kind)
    tu = sc.config.scaling.t_unit()
    t_r = t_g = 0.0
    t_end = sc.config.t_end / tu
    for k in range(1, 61):
        t_next = min(k * sc.config.dt_out / tu, t_end)
        t_r, dts_r, _ = ref.steps(t_r, t_next, 100_000, t_end=t_end)
        t_g, dts_g, _ = sim.steps(t_g, t_next, 100_000, t_end=t_end, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dts interval {k}")
        assert t_r == t_g
    assert t_g == t_end
    assert_bitwise(sim.state(), ref.state(), "four-side inflow state")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


def test_inflow_window_edges_bitwise(gpu, oracle_kind):
    """Inflow tiles take the safe-tile forms only while the stage's Mode-II ghost values are
    inside the window (tp_kernels.cu inflow_window_ok, checked on the device per stage).  A
    hydrograph that passes through depths and speeds far outside it (1e-35 m, 1e-33 m/s,
    phi 0 and 1, a 1e-31 m/s speed) alternates the inflow tiles between the safe and the
    checked forms: dt, state and audit stay bit-identical to the reference."""
    import dataclasses
    sc = scenarios.four_side_inflow(48, 40)
    samples = [(0.0, 1e-35, 0.6, 1e-33), (5.0, 2.0, 1.0, 3.0), (10.0, 1e-30, 0.0, 2.0),
               (15.0, 2.5, 0.5, 1e-31), (20.0, 0.0, 0.5, 0.0)]
    sc = dataclasses.replace(sc, hydrograph=dataclasses.replace(sc.hydrograph, samples=samples))
    sc.hydrograph.validate(sc.ncols, sc.nrows)
    ref, sim = _pair(sc, oracle_kind)
    tu = sc.config.scaling.t_unit()
    t_r = t_g = 0.0
    t_end = sc.config.t_end / tu
    for k in range(1, 61):
        t_next = min(k * sc.config.dt_out / tu, t_end)
        t_r, dts_r, _ = ref.steps(t_r, t_next, 100_000, t_end=t_end)
        t_g, dts_g, _ = sim.steps(t_g, t_next, 100_000, t_end=t_end, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dts interval {k}")
        assert t_r == t_g
    assert_bitwise(sim.state(), ref.state(), "inflow window-edge state")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-12, atol=1e-300)


def test_regularize_clips_small_negatives(gpu, oracle_kind):
    """regularize (solver.cpp:139-166): -1e-12 <= hp < 0 is clipped to 0 with its mass in the
    audit's 'clipped' slot, and the momenta of the now-dry phase are zeroed; then the run
    continues bit-identically."""
    sc = scenarios.wet_valley(40, 36)
    ref, sim = _pair(sc, oracle_kind)
    s = ref.state()
    rng = np.random.default_rng(5)
    for _ in range(30):
        f, j, i = int(rng.integers(0, 2)), int(rng.integers(3, 39)), int(rng.integers(3, 43))
        s[f, j, i] = -float(rng.uniform(1e-15, 9e-13))
    ref.set_state(s)
    sim.set_state(s)
    ref.reset_audit()
    sim.reset_audit()
    ref.regularize()
    sim.regularize()
    assert_bitwise(sim.state(), ref.state(), "after regularize")
    a_r, a_g = ref.audit(), sim.audit_array()
    assert a_r[4] != 0.0 and a_r[9] != 0.0
    np.testing.assert_allclose(a_g, a_r, rtol=1e-12, atol=1e-300)
    # the clipped slots are folded in the reference's (j, i) order (ClipList): bit for bit
    assert_bitwise(a_g[[4, 9]], a_r[[4, 9]], "clipped audit")
    tr, dts_r, _ = ref.steps(0.0, 1.0e9, 20, t_end=1.0e9)
    tg, dts_g, _ = sim.steps(0.0, 1.0e9, 20, t_end=1.0e9, record_dts=True)
    assert_bitwise(dts_g, dts_r, "dt sequence")
    assert_bitwise(sim.state(), ref.state(), "state after 20 steps")
    assert_bitwise(sim.audit_array()[[4, 9]], ref.audit()[[4, 9]], "clipped audit after 20 steps")


def test_clipped_audit_in_device_loop_bitwise(gpu, oracle_kind):
    """Small negative thicknesses planted in dry cells before each run are clipped by the
    stage kernels' regularize (predictor: -w, corrector: the Heun average -w/2) inside the
    device loop; the clipped slots of the audit match the reference's serial (j, i) sums bit
    for bit (ClipList, tp_types.h)."""
    sc = scenarios.c1_hill(72)
    ref, sim = _pair(sc, oracle_kind)
    rng = np.random.default_rng(11)
    t = 0.0
    for rnd in range(4):
        s = ref.state()
        dry = np.argwhere((s[0, 3:-3, 3:-3] == 0.0) & (s[1, 3:-3, 3:-3] == 0.0))
        for k in rng.choice(len(dry), 80, replace=False):
            j, i = dry[k] + 3
            s[int(rng.integers(0, 2)), j, i] = -float(rng.uniform(1e-15, 4e-13))
        ref.set_state(s)
        sim.set_state(s)
        tr, dts_r, _ = ref.steps(t, 1.0e9, 3, t_end=1.0e9)
        tg, dts_g, _ = sim.steps(t, 1.0e9, 3, t_end=1.0e9, record_dts=True)
        assert_bitwise(dts_g, dts_r, f"dt sequence, round {rnd}")
        assert tg == tr
        t = tr
        assert_bitwise(sim.state(), ref.state(), f"state, round {rnd}")
        a_r, a_g = ref.audit(), sim.audit_array()
        assert_bitwise(a_g[[4, 9]], a_r[[4, 9]], f"clipped audit, round {rnd}")
    assert a_r[4] != 0.0 and a_r[9] != 0.0


def _fuzz_scenario(seed):
    """A random small scenario: grid shape, terrain, release or four-side inflow, parameters."""
    from paper_2104_06784_b200.config import Hydrograph, SimConfig
    rng = np.random.default_rng(9000 + seed)
    nc, nr = int(rng.integers(3, 75)), int(rng.integers(2, 70))
    cs = float(rng.choice([1.0, 2.5, 5.0, 10.0]))
    z = scenarios.fractal_dem(nc, nr, cs, seed=int(rng.integers(1, 10_000)), relief=float(rng.uniform(5, 200)),
                              slope_deg=float(rng.uniform(0, 25)))
    inflow = bool(rng.integers(0, 2))
    cfg = SimConfig(mode="inflow" if inflow else "release", t_end=float(rng.uniform(5, 40)), dt_out=float(rng.uniform(0.3, 3)))
    p = cfg.params
    p.delta_b, p.C_d, p.N_R = float(rng.uniform(5, 35)), float(rng.uniform(0, 10)), float(rng.uniform(20, 800))
    p.theta_b, p.phi_s0, p.alpha_rho = float(rng.uniform(0, 10)), float(rng.uniform(0.2, 0.8)), float(rng.uniform(0.2, 1.0))
    cfg.cfl = float(rng.uniform(0.05, 0.125))
    if inflow:
        cells = []
        for side in ("W", "E", "S", "N"):
            if rng.integers(0, 2):
                n_side = nr if side in "WE" else nc
                a = int(rng.integers(0, n_side))
                b = min(n_side, a + int(rng.integers(1, 6)))
                for k in range(a, b):
                    cells.append({"W": (0, k, "W"), "E": (nc - 1, k, "E"), "S": (k, 0, "S"), "N": (k, nr - 1, "N")}[side])
        if not cells:
            cells = [(0, 0, "W")]
        t1 = float(rng.uniform(2, 20))
        samples = [(0.0, float(rng.uniform(0, 1)), 0.5, 1.0), (t1, float(rng.uniform(0.5, 4)), float(rng.uniform(0.3, 0.7)),
                                                               float(rng.uniform(0, 6))), (2 * t1, 0.0, 0.5, 0.0)]
        return scenarios.Scenario(f"fuzz{seed}", z, cs, cfg, hydrograph=Hydrograph(cells=cells, samples=samples))
    h0 = scenarios.paraboloid_release(nc, nr, h0=float(rng.uniform(0.5, 10)), rx=max(1.0, nc * rng.uniform(0.1, 0.5)),
                                      ry=max(1.0, nr * rng.uniform(0.1, 0.5)), cx=nc * rng.uniform(0.2, 0.8),
                                      cy=nr * rng.uniform(0.2, 0.8))
    return scenarios.Scenario(f"fuzz{seed}", z, cs, cfg, h0=h0)


@pytest.mark.parametrize("seed", list(range(40)))
def test_fuzz_scenarios_bitwise(gpu, oracle_kind, seed):
    """Random small scenarios (shape, terrain, release or inflow on random sides, parameters)
    through the run loop's output schedule: every dt and the final state bit-identical."""
    sc = _fuzz_scenario(seed)
    ref, sim = _pair(sc, oracle_kind, wide=None if seed % 2 == 0 else False)  # odd seeds: production CTAs
    tu = sc.config.scaling.t_unit()
    t_end, dt_out = sc.config.t_end / tu, sc.config.dt_out / tu
    t_r = t_g = 0.0
    k, done = 1, 0
    from oracle.oracle import OracleError
    while done < 150 and t_r < t_end:
        t_next = min(k * dt_out, t_end)
        try:
            t_r, dts_r, hit_r = ref.steps(t_r, t_next, 150 - done, t_end=t_end)
        except OracleError as er:  # the reference itself stops (e.g. regularize): same error here
            with pytest.raises(NumericsError) as eg:
                sim.steps(t_g, t_next, 150 - done, t_end=t_end)
            assert str(eg.value) == str(er)
            return
        t_g, dts_g, hit_g = sim.steps(t_g, t_next, 150 - done, t_end=t_end, record_dts=True)
        assert_bitwise(np.asarray(dts_g), np.asarray(dts_r), f"dts interval {k}")
        assert t_r == t_g
        done += len(dts_r)
        if hit_r:
            k += 1
    assert_bitwise(sim.state(), ref.state(), f"state ({sc.ncols}x{sc.nrows}, {sc.config.mode})")
    np.testing.assert_allclose(sim.audit_array(), ref.audit(), rtol=1e-11, atol=1e-300)
