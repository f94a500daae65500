"""`Simulator` — the reference's solver API on the B200 path.

Mirrors ``tpflow::Simulator`` (/root/reference/proj/include/tpflow/solver.hpp:26-98)
method for method, with the same argument meaning (scaled times for the step
pieces, physical units for inputs/outputs) and the same exceptions
(ConfigError/IoError/NumericsError, errors.hpp:8-21).  All numerics run in the
sm_100a kernels behind the C ABI (include/tpflow_b200.h); this class only
marshals host arrays and reproduces ``Simulator::run``'s host loop
(solver.cpp:619-659), whose inner steps run device-resident (tp_steps).
"""
from __future__ import annotations

import ctypes as C
import time
from typing import Callable, Optional

import numpy as np

from . import _lib
from .config import (ERRORS_BY_CODE, Hydrograph, MassAudit, RunReport, SimConfig, TpflowError)

KGHOST = 3  # solver.hpp:14


class CudaError(TpflowError):
    exit_code = 5


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def make_params(cfg: SimConfig, device: int = 0) -> _lib.TpParams:
    p = cfg.params
    s = cfg.scaling
    return _lib.TpParams(p.delta_b, p.C_d, p.N_R, p.theta_b, p.phi_s0, p.alpha_rho, p.chi,
                         s.L, s.H, s.g, cfg.t_end, cfg.dt_out, cfg.cfl, cfg.h_dry, cfg.eps_h,
                         1 if cfg.inflow else 0, device)


class SimSnapshot:
    """config.hpp:48-56 — interior fields in physical units."""

    def __init__(self, t: float, step_index: int, fields: np.ndarray):
        self.t = t
        self.step_index = step_index
        self.h_total, self.phi_s, self.vX_s, self.vY_s, self.vX_f, self.vY_f = fields


class Simulator:
    """One device-resident simulation (optionally a row slab [row0, row1) of the DEM)."""

    def __init__(self, config: SimConfig, z: np.ndarray, cellsize: float, xll: float = 0.0,
                 yll: float = 0.0, device: int = 0, rows: Optional[tuple] = None,
                 fastdiv: bool = True):
        self.L = _lib.lib()
        self.cfg = config
        z = np.ascontiguousarray(z, dtype=np.float64)
        self._z = z
        self.nrows_g, self.ncols = z.shape
        self._params = make_params(config, device)
        self._dem = _lib.TpDem(self.ncols, self.nrows_g, xll, yll, cellsize, _dp(z))
        h = C.c_void_p()
        if rows is None:
            rc = self.L.tp_create(C.byref(self._params), C.byref(self._dem), C.byref(h))
            self.row0, self.row1 = 0, self.nrows_g
        else:
            self.row0, self.row1 = rows
            rc = self.L.tp_create_slab(C.byref(self._params), C.byref(self._dem), self.row0,
                                       self.row1, C.byref(h))
        self.h = h
        self._check(rc)
        nx, ny, dxi, deta = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        self._check(self.L.tp_dims(h, C.byref(nx), C.byref(ny), C.byref(dxi), C.byref(deta)))
        self.nx, self.ny, self.dxi, self.deta = nx.value, ny.value, dxi.value, deta.value
        self.nrows = self.row1 - self.row0
        if not fastdiv:
            self.set_option("fastdiv", 0)
        self._hydro: Optional[Hydrograph] = None

    @classmethod
    def from_scenario(cls, sc, device: int = 0, rows=None, fastdiv: bool = True, init: bool = True):
        sim = cls(sc.config, sc.z, sc.cellsize, sc.xll, sc.yll, device=device, rows=rows, fastdiv=fastdiv)
        if init:
            if sc.h0 is not None:
                sim.set_initial_thickness(sc.h0)
                if sc.vx0 is not None:
                    sim.set_initial_velocity(sc.vx0, sc.vy0)
            if sc.hydrograph is not None:
                sim.set_hydrograph(sc.hydrograph)
        return sim

    # -- plumbing -------------------------------------------------------------------
    def _check(self, rc: int) -> None:
        if rc != 0:
            msg = self.L.tp_last_error(self.h).decode() if self.h else "tp_create failed"
            raise ERRORS_BY_CODE.get(rc, CudaError if rc == 5 else TpflowError)(msg)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.L.tp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: str, value: int) -> None:
        self._check(self.L.tp_set_option(self.h, key.encode(), int(value)))

    # -- setup (solver.cpp:35-81) ------------------------------------------------------
    def set_initial_thickness(self, h_m: np.ndarray) -> None:
        h_m = np.ascontiguousarray(h_m, dtype=np.float64)
        if h_m.shape != (self.nrows_g, self.ncols):
            raise ERRORS_BY_CODE[2](
                f"initial state: dimension mismatch with DEM ({h_m.shape[1]}x{h_m.shape[0]} vs "
                f"{self.ncols}x{self.nrows_g})")
        self._check(self.L.tp_set_initial_thickness(self.h, _dp(h_m)))

    def set_initial_velocity(self, vx: np.ndarray, vy: np.ndarray) -> None:
        vx = np.ascontiguousarray(vx, dtype=np.float64)
        vy = np.ascontiguousarray(vy, dtype=np.float64)
        if vx.shape != (self.nrows_g, self.ncols) or vx.shape != vy.shape:
            raise ERRORS_BY_CODE[2]("initial velocity: dimension mismatch with DEM")
        self._check(self.L.tp_set_initial_velocity(self.h, _dp(vx), _dp(vy)))

    def set_hydrograph(self, hg: Hydrograph) -> None:
        ci = np.array([c[0] for c in hg.cells], dtype=np.int32)
        cj = np.array([c[1] for c in hg.cells], dtype=np.int32)
        side = "".join(c[2] for c in hg.cells).encode()
        s = np.array(hg.samples, dtype=np.float64).reshape(-1, 4)
        cols = [np.ascontiguousarray(s[:, k]) for k in range(4)]
        ip = C.POINTER(C.c_int)
        self._check(self.L.tp_set_hydrograph(self.h, len(ci), ci.ctypes.data_as(ip),
                                             cj.ctypes.data_as(ip), side, len(s),
                                             *[_dp(c) for c in cols]))
        self._hydro = hg

    # -- state / geometry -------------------------------------------------------------
    def state(self) -> np.ndarray:
        out = np.empty((6, self.ny, self.nx))
        self._check(self.L.tp_get_state(self.h, _dp(out)))
        return out

    def set_state(self, s: np.ndarray) -> None:
        s = np.ascontiguousarray(s, dtype=np.float64)
        assert s.shape == (6, self.ny, self.nx), s.shape
        self._check(self.L.tp_set_state(self.h, _dp(s)))

    def geometry(self) -> np.ndarray:
        out = np.empty((14, self.ny, self.nx))
        self._check(self.L.tp_get_geometry(self.h, _dp(out)))
        return out

    # -- the step pieces (solver.hpp:41-47) ------------------------------------------------
    def apply_boundaries(self, t_scaled: float) -> None:
        self._check(self.L.tp_apply_boundaries(self.h, t_scaled))

    def compute_dt(self, t_scaled: float, t_next_scaled: float) -> float:
        dt = C.c_double()
        self._check(self.L.tp_compute_dt(self.h, t_scaled, t_next_scaled, C.byref(dt)))
        return dt.value

    def advance_step(self, dt_scaled: float, t_scaled: float) -> None:
        self._check(self.L.tp_advance_step(self.h, dt_scaled, t_scaled))

    def regularize(self) -> None:
        self._check(self.L.tp_regularize(self.h))

    def set_advection_only(self, on: bool) -> None:
        self._check(self.L.tp_set_advection_only(self.h, 1 if on else 0))

    def steps(self, t: float, t_next: float, max_steps: int, t_end: Optional[float] = None,
              record_dts: bool = False):
        """Device-resident loop body of Simulator::run (solver.cpp:637-649).  Returns (t, dts|n, hit)."""
        tt = C.c_double(t)
        n = C.c_long()
        hit = C.c_int()
        te = t_next if t_end is None else t_end
        dts = np.zeros(max(1, max_steps)) if record_dts else None
        self._check(self.L.tp_steps(self.h, t_next, te, int(max_steps), C.byref(tt), C.byref(n),
                                    C.byref(hit), _dp(dts) if record_dts else None))
        return tt.value, (dts[: n.value].copy() if record_dts else n.value), bool(hit.value)

    def set_stream(self, cuda_stream_handle: int) -> None:
        """Launch on an external CUDA stream (e.g. torch.cuda.Stream().cuda_stream)."""
        self._check(self.L.tp_set_stream(self.h, C.c_void_p(cuda_stream_handle)))

    def kernel_launches(self) -> int:
        return int(self.L.tp_kernel_launches(self.h))

    def active_tiles(self) -> tuple:
        """(predictor, corrector) tiles processed by the last step, and the grid's tile count."""
        p, c, t = C.c_int(), C.c_int(), C.c_int()
        self._check(self.L.tp_active_tiles(self.h, C.byref(p), C.byref(c), C.byref(t)))
        return p.value, c.value, t.value

    def safe_tiles(self) -> int:
        """Tiles of the last corrector list that ran the safe (window-test-free) path."""
        n = C.c_int()
        self._check(self.L.tp_safe_tiles(self.h, C.byref(n)))
        return n.value

    def synchronize(self) -> None:
        self._check(self.L.tp_synchronize(self.h))

    # -- audit / mass / snapshot --------------------------------------------------------
    def _audit(self) -> np.ndarray:
        a = np.zeros(10)
        self._check(self.L.tp_get_audit(self.h, _dp(a)))
        return a

    def _set_audit(self, a: np.ndarray) -> None:
        a = np.ascontiguousarray(a, dtype=np.float64)
        self._check(self.L.tp_set_audit(self.h, _dp(a)))

    def solid_audit(self) -> MassAudit:
        return MassAudit(*self._audit()[0:5])

    def fluid_audit(self) -> MassAudit:
        return MassAudit(*self._audit()[5:10])

    def audit_array(self) -> np.ndarray:
        return self._audit()

    def reset_audit(self) -> None:
        self._set_audit(np.zeros(10))

    def interior_mass(self):
        ms, mf = C.c_double(), C.c_double()
        self._check(self.L.tp_interior_mass(self.h, C.byref(ms), C.byref(mf)))
        return ms.value, mf.value

    def interior_mass_device(self):
        """(solid, fluid) interior masses reduced on the device (within ~1 ulp of exact)."""
        ms, mf = C.c_double(), C.c_double()
        self._check(self.L.tp_interior_mass_device(self.h, C.byref(ms), C.byref(mf)))
        return ms.value, mf.value

    def interior_mass_solid(self) -> float:
        return self.interior_mass()[0]

    def interior_mass_fluid(self) -> float:
        return self.interior_mass()[1]

    def snapshot(self, t_scaled: float, step_index: int = 0) -> SimSnapshot:
        out = np.empty((6, self.nrows, self.ncols))
        self._check(self.L.tp_snapshot(self.h, _dp(out)))
        return SimSnapshot(t_scaled * self.cfg.scaling.t_unit(), step_index, out)

    # -- the run loop (solver.cpp:619-659) ----------------------------------------------
    def run(self, sink: Optional[Callable[[SimSnapshot], None]] = None,
            max_steps: Optional[int] = None) -> RunReport:
        report = RunReport()
        self.reset_audit()
        self.regularize()
        a = self._audit()
        ms, mf = self.interior_mass()
        a[0], a[5] = ms, mf
        self._set_audit(a)

        t_unit = self.cfg.scaling.t_unit()
        t_end = self.cfg.t_end / t_unit
        dt_out = self.cfg.dt_out / t_unit
        t = 0.0
        steps = 0
        if sink:
            sink(self.snapshot(t, steps))
        next_out = dt_out
        budget = max_steps if max_steps is not None else (1 << 62)

        t0 = time.perf_counter()
        while t < t_end and steps < budget:
            t_next = min(next_out, t_end)
            t, n, hit = self.steps(t, t_next, budget - steps, t_end=t_end)
            steps += n
            if hit:
                if sink:
                    sink(self.snapshot(t, steps))
                if t_next == next_out:
                    next_out += dt_out
        t1 = time.perf_counter()

        report.steps = steps
        report.wall_seconds = t1 - t0
        a = self._audit()
        ms, mf = self.interior_mass()
        a[1], a[6] = ms, mf
        self._set_audit(a)
        report.solid = MassAudit(*a[0:5])
        report.fluid = MassAudit(*a[5:10])
        return report
