"""The CPU oracle itself (no GPU): the C restatement (oracle/tpflow_oracle.c) is
pinned bit for bit to the unmodified reference compiled in place (oracle/_ref),
and both to the SPEC.md known-answer values.  These run in the CPU suite."""
import math
import os

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2104_06784_b200 import scenarios
from tests.util import assert_bitwise

HAVE_REF = orc.available("ref") or os.path.exists(orc.REF_SOURCES)
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built and /root/reference absent")


def _pair(sc):
    return orc.OracleSim(sc, "ref"), orc.OracleSim(sc, "port")


@needs_ref
@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(40), lambda: scenarios.c4_terrain(50, 36),
                                  lambda: scenarios.c3_channel(64, 32)])
def test_port_geometry_and_state_bitwise(make):
    sc = make()
    ref, port = _pair(sc)
    assert_bitwise(port.geometry(), ref.geometry(), "geometry")
    assert_bitwise(port.state(), ref.state(), "initial state")


@needs_ref
def test_port_step_pieces_bitwise():
    sc = scenarios.c1_hill(40)
    ref, port = _pair(sc)
    t = 0.0
    for n in range(6):
        ref.apply_boundaries(t)
        port.apply_boundaries(t)
        assert_bitwise(port.state(), ref.state(), f"bc {n}")
        d_r, d_p = ref.compute_dt(t, 1e9), port.compute_dt(t, 1e9)
        assert d_r == d_p
        ref.advance_step(d_r, t)
        port.advance_step(d_r, t)
        assert_bitwise(port.state(), ref.state(), f"advance {n}")
        t += d_r
    np.testing.assert_array_equal(port.audit(), ref.audit())


@needs_ref
@pytest.mark.parametrize("make,steps", [(lambda: scenarios.c1_hill(48), 120),
                                        (lambda: scenarios.c3_channel(64, 32, t_end=20.0, dt_out=0.5), 200),
                                        (lambda: scenarios.wet_valley(40, 36), 60)])
def test_port_trajectory_bitwise(make, steps):
    sc = make()
    ref, port = _pair(sc)
    tu = sc.config.scaling.t_unit()
    t_next = 0.5 / tu if sc.config.inflow else 1e9
    t_r = t_p = 0.0
    done = 0
    while done < steps:
        t_r, d_r, _ = ref.steps(t_r, t_next, steps - done, t_end=1e9)
        t_p, d_p, _ = port.steps(t_p, t_next, steps - done, t_end=1e9)
        assert_bitwise(d_p, d_r, "dts")
        assert t_r == t_p
        done += len(d_r)
        t_next += 0.5 / tu
    assert_bitwise(port.state(), ref.state(), "trajectory state")
    np.testing.assert_array_equal(port.audit(), ref.audit())
    assert port.interior_mass() == ref.interior_mass()


@needs_ref
def test_port_run_and_errors_match():
    sc = scenarios.c1_hill(32, t_end=2.0, dt_out=0.5)
    ref, port = _pair(sc)
    rr, sr = ref.run()
    rp, sp = port.run()
    assert rr[0] == rp[0]
    np.testing.assert_array_equal(sr, sp)
    np.testing.assert_array_equal(rr[2:], rp[2:])
    # NumericsError text (solver.cpp:147-152)
    s = ref.state()
    s[1, 9, 11] = -3e-9
    for o in (ref, port):
        o.set_state(s)
    msgs = []
    for o in (ref, port):
        with pytest.raises(orc.OracleError) as e:
            o.regularize()
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] and "negative fluid thickness" in msgs[0]


def test_port_known_answers_spec():
    """SPEC.md worked examples through the port's step pieces (no reference needed)."""
    from paper_2104_06784_b200.scenarios import Scenario
    from paper_2104_06784_b200.config import SimConfig
    # geometry: 30 degree plane -> n = (-0.5, 0, 0.8660), J_b = 1.1547
    n = 12
    x = (np.arange(n) + 0.5) * 1.0
    z = np.tile(x * math.tan(math.radians(30.0)), (n, 1))
    sc = Scenario("plane30", z, 1.0, SimConfig(mode="release", t_end=1.0, dt_out=1.0), h0=np.zeros((n, n)))
    g = orc.OracleSim(sc, "port").geometry()
    c = (slice(3, -3), slice(3, -3))
    np.testing.assert_allclose(g[0][c], -0.5, atol=1e-4)
    np.testing.assert_allclose(g[1][c], 0.0, atol=1e-12)
    np.testing.assert_allclose(g[2][c], 0.8660, atol=1e-4)
    np.testing.assert_allclose(g[3][c], 1.1547, atol=1e-4)
    np.testing.assert_allclose(g[3] * g[2], 1.0, atol=1e-12)  # J_b * c == 1
    # flat terrain: n = (0,0,1), J_b = 1, A = I
    sc2 = Scenario("flat", np.full((n, n), 5.0), 1.0, SimConfig(mode="release", t_end=1.0, dt_out=1.0),
                   h0=np.ones((n, n)))
    o = orc.OracleSim(sc2, "port")
    g2 = o.geometry()
    for k, v in ((0, 0.0), (1, 0.0), (2, 1.0), (3, 1.0), (4, 1.0), (5, 0.0), (6, 0.0), (7, 1.0)):
        np.testing.assert_array_equal(g2[k], v)
    # compute_dt: v=0, h=1, c=1, eps=1 -> lambda = 1 -> dt = cfl*dx/1
    assert o.compute_dt(0.0, 1e9) == 0.1 * 1.0 / 1.0
    # all-dry domain -> dt = remaining
    sc3 = Scenario("dry", np.zeros((n, n)), 1.0, SimConfig(mode="release", t_end=1.0, dt_out=1.0),
                   h0=np.zeros((n, n)))
    assert orc.OracleSim(sc3, "port").compute_dt(0.25, 0.8) == 0.8 - 0.25
    # quiescence: uniform wet state on flat terrain stays put
    t = 0.0
    s0 = o.state()
    for _ in range(20):
        o.apply_boundaries(t)
        dt = o.compute_dt(t, 1e9)
        o.advance_step(dt, t)
        t += dt
    np.testing.assert_allclose(o.state()[:, 3:-3, 3:-3], s0[:, 3:-3, 3:-3], atol=1e-14)


def test_reduce_max_spec():
    """Backend::reduce_max examples: exact max, ghosts of zero."""
    v = np.array([0.0, 3.0, 1.5, 7.25, 2.0])
    assert orc.reduce_max(v, kind="port") == 7.25
    if HAVE_REF:
        assert orc.reduce_max(v, kind="ref", lanes=4) == 7.25
        assert orc.reduce_max(v, kind="ref") == 7.25
