"""TEST INFRASTRUCTURE ONLY — the CPU checker.

ctypes front-end for the two CPU implementations of the reference step API:

* ``kind="ref"``  — oracle/_ref/libtpflow_ref.so, the UNMODIFIED reference
  (/root/reference/proj/src/*.cpp) compiled in place by oracle/Makefile, driven
  through the shim in oracle/ref_harness.cpp;
* ``kind="port"`` — oracle/_port/libtpflow_oracle.so, the plain-C restatement in
  oracle/tpflow_oracle.c (same entry points, prefix ``orc_``), which also runs on
  row slabs for the multi-rank tests.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import this.
The product path (paper_2104_06784_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "libtpflow_ref.so")
PORT_SO = os.path.join(HERE, "_port", "libtpflow_oracle.so")
REF_SOURCES = "/root/reference/proj/src/solver.cpp"


class _Params(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "delta_b", "C_d", "N_R", "theta_b", "phi_s0", "alpha_rho", "chi",
        "L", "H", "g", "t_end", "dt_out", "cfl", "h_dry", "eps_h")] + [
        ("mode", C.c_int), ("lanes", C.c_int)]


def build(kind: str = "all") -> None:
    """Build the checkers (make -C oracle).  The ref target needs /root/reference."""
    target = {"all": "all", "ref": "ref", "port": "port"}[kind]
    subprocess.run(["make", "-s", "-C", HERE, target], check=True)


def available(kind: str) -> bool:
    return os.path.exists(REF_SO if kind == "ref" else PORT_SO)


_LIBS = {}


def _lib(kind: str):
    if kind in _LIBS:
        return _LIBS[kind]
    path = REF_SO if kind == "ref" else PORT_SO
    if not os.path.exists(path):
        if kind == "ref" and not os.path.exists(REF_SOURCES):
            raise FileNotFoundError(f"{path} missing and /root/reference absent")
        build(kind)
    lib = C.CDLL(path)
    p = "ref_" if kind == "ref" else "orc_"
    vp, dp, ip, lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_long)

    def fn(name, res, *args):
        f = getattr(lib, p + name)
        f.restype = res
        f.argtypes = list(args)
        return f

    lib.f = {
        "create": fn("create", C.c_int, C.POINTER(_Params), C.c_int, C.c_int, C.c_double, C.c_double,
                     C.c_double, dp, C.POINTER(vp)),
        "destroy": fn("destroy", None, vp),
        "last_error": fn("last_error", C.c_char_p, vp),
        "dims": fn("dims", None, vp, ip, ip, dp, dp),
        "set_initial_thickness": fn("set_initial_thickness", C.c_int, vp, dp),
        "set_initial_velocity": fn("set_initial_velocity", C.c_int, vp, dp, dp),
        "set_hydrograph": fn("set_hydrograph", C.c_int, vp, C.c_int, ip, ip, C.c_char_p, C.c_int,
                             dp, dp, dp, dp),
        "get_state": fn("get_state", None, vp, dp),
        "set_state": fn("set_state", None, vp, dp),
        "get_geometry": fn("get_geometry", None, vp, dp),
        "apply_boundaries": fn("apply_boundaries", C.c_int, vp, C.c_double),
        "compute_dt": fn("compute_dt", C.c_int, vp, C.c_double, C.c_double, dp),
        "advance_step": fn("advance_step", C.c_int, vp, C.c_double, C.c_double),
        "regularize": fn("regularize", C.c_int, vp),
        "set_advection_only": fn("set_advection_only", None, vp, C.c_int),
        "get_audit": fn("get_audit", None, vp, dp),
        "reset_audit": fn("reset_audit", None, vp),
        "interior_mass": fn("interior_mass", None, vp, dp, dp),
        "steps": fn("steps", C.c_int, vp, C.c_double, C.c_double, C.c_long, dp, lp, ip, dp),
        "run": fn("run", C.c_int, vp, dp, dp, C.c_int, ip),
        "snapshot": fn("snapshot", None, vp, C.c_double, dp),
    }
    lib.f["reduce_max"] = fn("reduce_max", C.c_int, C.c_int, dp, C.c_long, dp)
    _LIBS[kind] = lib
    return lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class OracleSim:
    """One reference ``Simulator`` (or its C restatement) on a scenario."""

    def __init__(self, scenario, kind: str = "ref", lanes: int = 0, init: bool = True):
        self.kind = kind
        self.lib = _lib(kind)
        self.f = self.lib.f
        cfg = scenario.config
        p = _Params(cfg.params.delta_b, cfg.params.C_d, cfg.params.N_R, cfg.params.theta_b,
                    cfg.params.phi_s0, cfg.params.alpha_rho, cfg.params.chi,
                    cfg.scaling.L, cfg.scaling.H, cfg.scaling.g,
                    cfg.t_end, cfg.dt_out, cfg.cfl, cfg.h_dry, cfg.eps_h,
                    1 if cfg.inflow else 0, lanes)
        self.ncols, self.nrows = scenario.ncols, scenario.nrows
        z = np.ascontiguousarray(scenario.z, dtype=np.float64)
        h = C.c_void_p()
        rc = self.f["create"](C.byref(p), self.ncols, self.nrows, scenario.cellsize,
                              scenario.xll, scenario.yll, _dp(z), C.byref(h))
        self.h = h
        self._check(rc)
        nx, ny, dxi, deta = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        self.f["dims"](h, C.byref(nx), C.byref(ny), C.byref(dxi), C.byref(deta))
        self.nx, self.ny, self.dxi, self.deta = nx.value, ny.value, dxi.value, deta.value
        self.t_unit = cfg.scaling.t_unit()
        if init:
            if scenario.h0 is not None:
                self._check(self.f["set_initial_thickness"](h, _dp(np.ascontiguousarray(scenario.h0))))
                if scenario.vx0 is not None:
                    self._check(self.f["set_initial_velocity"](
                        h, _dp(np.ascontiguousarray(scenario.vx0)), _dp(np.ascontiguousarray(scenario.vy0))))
            if scenario.hydrograph is not None:
                self.set_hydrograph(scenario.hydrograph)

    def __del__(self):
        try:
            if self.h:
                self.f["destroy"](self.h)
        except Exception:
            pass

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.f["last_error"](self.h).decode())

    def set_hydrograph(self, hg):
        n = len(hg.cells)
        ci = np.array([c[0] for c in hg.cells], dtype=np.int32)
        cj = np.array([c[1] for c in hg.cells], dtype=np.int32)
        side = "".join(c[2] for c in hg.cells).encode()
        s = np.array(hg.samples, dtype=np.float64).reshape(-1, 4)
        cols = [np.ascontiguousarray(s[:, k]) for k in range(4)]
        ip = C.POINTER(C.c_int)
        self._check(self.f["set_hydrograph"](self.h, n, ci.ctypes.data_as(ip), cj.ctypes.data_as(ip),
                                             side, len(s), *[_dp(c) for c in cols]))

    # --- state / geometry ------------------------------------------------------
    def state(self) -> np.ndarray:
        out = np.empty((6, self.ny, self.nx))
        self.f["get_state"](self.h, _dp(out))
        return out

    def set_state(self, s: np.ndarray) -> None:
        s = np.ascontiguousarray(s, dtype=np.float64)
        assert s.shape == (6, self.ny, self.nx)
        self.f["set_state"](self.h, _dp(s))

    def geometry(self) -> np.ndarray:
        out = np.empty((14, self.ny, self.nx))
        self.f["get_geometry"](self.h, _dp(out))
        return out

    # --- step API (solver.hpp:41-47) ---------------------------------------------
    def apply_boundaries(self, t: float) -> None:
        self._check(self.f["apply_boundaries"](self.h, t))

    def compute_dt(self, t: float, t_next: float) -> float:
        dt = C.c_double()
        self._check(self.f["compute_dt"](self.h, t, t_next, C.byref(dt)))
        return dt.value

    def advance_step(self, dt: float, t: float) -> None:
        self._check(self.f["advance_step"](self.h, dt, t))

    def regularize(self) -> None:
        self._check(self.f["regularize"](self.h))

    def set_advection_only(self, on: bool) -> None:
        self.f["set_advection_only"](self.h, 1 if on else 0)

    def audit(self) -> np.ndarray:
        a = np.empty(10)
        self.f["get_audit"](self.h, _dp(a))
        return a

    def reset_audit(self) -> None:
        self.f["reset_audit"](self.h)

    def interior_mass(self):
        ms, mf = C.c_double(), C.c_double()
        self.f["interior_mass"](self.h, C.byref(ms), C.byref(mf))
        return ms.value, mf.value

    def steps(self, t: float, t_next: float, max_steps: int, t_end: float = None):
        """Simulator::run's loop body (solver.cpp:637-649) from scaled time t.

        Returns (t, dts, hit)."""
        tt = C.c_double(t)
        n = C.c_long()
        hit = C.c_int()
        dts = np.zeros(max(1, max_steps))
        te = t_next if t_end is None else t_end
        self._check(self.f["steps"](self.h, t_next, te, max_steps, C.byref(tt), C.byref(n),
                                    C.byref(hit), _dp(dts)))
        return tt.value, dts[: n.value].copy(), bool(hit.value)

    def run(self, max_snaps: int = 4096):
        rep = np.zeros(12)
        snaps = np.zeros(max_snaps)
        n = C.c_int()
        self._check(self.f["run"](self.h, _dp(rep), _dp(snaps), max_snaps, C.byref(n)))
        return rep, snaps[: min(n.value, max_snaps)].copy()

    def snapshot(self, t: float) -> np.ndarray:
        out = np.empty((6, self.nrows, self.ncols))
        self.f["snapshot"](self.h, t, _dp(out))
        return out


class OracleSlab:
    """A row slab of the C restatement with the split-step interface of
    paper_2104_06784_b200.distributed.CudaSlab (tests: gloo / in-process runs)."""

    def __init__(self, scenario, rows, lanes: int = 0):
        import torch
        lib = _lib("port")
        L = lib
        vp, dp, ip = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int)
        for name, res, args in [
            ("orc_create_slab", C.c_int, [C.POINTER(_Params), C.c_int, C.c_int, C.c_double, C.c_double,
                                          C.c_double, dp, C.c_int, C.c_int, C.POINTER(vp)]),
            ("orc_halo_doubles", C.c_long, [vp]), ("orc_halo_pack", None, [vp, C.c_int, C.c_int, dp]),
            ("orc_halo_unpack", None, [vp, C.c_int, C.c_int, dp]),
            ("orc_step_begin", None, [vp, C.c_double, C.c_double, C.c_double]), ("orc_bc", None, [vp, C.c_int]),
            ("orc_lambda_local", C.c_double, [vp]), ("orc_dt_from", None, [vp, C.c_double]),
            ("orc_stage", C.c_int, [vp, C.c_int]), ("orc_step_end", C.c_int, [vp, dp, ip, dp])]:
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        self.L = L
        cfg = scenario.config
        p = _Params(cfg.params.delta_b, cfg.params.C_d, cfg.params.N_R, cfg.params.theta_b,
                    cfg.params.phi_s0, cfg.params.alpha_rho, cfg.params.chi,
                    cfg.scaling.L, cfg.scaling.H, cfg.scaling.g,
                    cfg.t_end, cfg.dt_out, cfg.cfl, cfg.h_dry, cfg.eps_h, 1 if cfg.inflow else 0, lanes)
        z = np.ascontiguousarray(scenario.z, dtype=np.float64)
        h = C.c_void_p()
        self.row0, self.row1 = rows
        rc = L.orc_create_slab(C.byref(p), scenario.ncols, scenario.nrows, scenario.cellsize, 0.0, 0.0,
                               _dp(z), self.row0, self.row1, C.byref(h))
        self.h = h
        if rc:
            raise OracleError(rc, L.f["last_error"](h).decode())
        if scenario.h0 is not None:
            self._ck(L.f["set_initial_thickness"](h, _dp(np.ascontiguousarray(scenario.h0))))
        if scenario.hydrograph is not None:
            hg = scenario.hydrograph
            ci = np.array([c[0] for c in hg.cells], dtype=np.int32)
            cj = np.array([c[1] for c in hg.cells], dtype=np.int32)
            sd = "".join(c[2] for c in hg.cells).encode()
            smp = np.array(hg.samples, dtype=np.float64).reshape(-1, 4)
            cols = [np.ascontiguousarray(smp[:, k]) for k in range(4)]
            self._ck(L.f["set_hydrograph"](h, len(ci), ci.ctypes.data_as(ip), cj.ctypes.data_as(ip), sd,
                                           len(smp), *[_dp(c) for c in cols]))
        n = int(L.orc_halo_doubles(h))
        self.send = [torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)]
        self.recv = [torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)]
        nx, ny, dxi, deta = C.c_int(), C.c_int(), C.c_double(), C.c_double()
        L.f["dims"](h, C.byref(nx), C.byref(ny), C.byref(dxi), C.byref(deta))
        self.nx, self.ny = nx.value, ny.value

    def _ck(self, rc):
        if rc:
            raise OracleError(rc, self.L.f["last_error"](self.h).decode())

    @staticmethod
    def _tp(t):
        return C.cast(t.data_ptr(), C.POINTER(C.c_double))

    def pack(self, buf, side):
        self.L.orc_halo_pack(self.h, buf, side, self._tp(self.send[side]))
        return self.send[side]

    def unpack(self, buf, side, src=None):
        src = self.recv[side] if src is None else src
        self.L.orc_halo_unpack(self.h, buf, side, self._tp(src.contiguous()))

    def step_begin(self, t, t_next, t_end):
        self.L.orc_step_begin(self.h, t, t_next, t_end)

    def bc(self, buf):
        self.L.orc_bc(self.h, buf)

    def lambda_local(self):
        return float(self.L.orc_lambda_local(self.h))

    def dt_from(self, lam):
        self.L.orc_dt_from(self.h, float(lam))

    def stage(self, corrector):
        self._ck(self.L.orc_stage(self.h, corrector))

    def step_end(self):
        t, hit, dt = C.c_double(), C.c_int(), C.c_double()
        self._ck(self.L.orc_step_end(self.h, C.byref(t), C.byref(hit), C.byref(dt)))
        return t.value, bool(hit.value), dt.value

    def state(self):
        out = np.empty((6, self.ny, self.nx))
        self.L.f["get_state"](self.h, _dp(out))
        return out

    def audit(self):
        a = np.empty(10)
        self.L.f["get_audit"](self.h, _dp(a))
        return a

    def __del__(self):
        try:
            self.L.f["destroy"](self.h)
        except Exception:
            pass


def reduce_max(values: np.ndarray, lanes: int = 0, kind: str = "ref") -> float:
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = C.c_double()
    rc = _lib(kind).f["reduce_max"](lanes, _dp(v), v.size, C.byref(out))
    if rc != 0:
        raise OracleError(rc, "reduce_max: empty input")
    return out.value
