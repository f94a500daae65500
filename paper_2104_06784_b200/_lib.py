"""ctypes binding of the C ABI (include/tpflow_b200.h) — the product path.

Loads the in-tree ``paper_2104_06784_b200/libtpflow_b200.so`` (built by
``__graft_entry__.build()`` / ``make -C paper_2104_06784_b200/csrc``).  There is
no fallback: if the library or a CUDA device is missing, every entry point
raises.  This is the same binding a maintainer would add to the reference's
Python tooling.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtpflow_b200.so")
# development override (e.g. the `make timing` probe build); the product path is LIB_PATH
LIB_PATH = os.environ.get("TPFLOW_B200_LIB", LIB_PATH)
CSRC = os.path.join(HERE, "csrc")


class TpParams(C.Structure):
    _fields_ = [(n, C.c_double) for n in (
        "delta_b", "C_d", "N_R", "theta_b", "phi_s0", "alpha_rho", "chi",
        "L", "H", "g", "t_end", "dt_out", "cfl", "h_dry", "eps_h")] + [
        ("mode", C.c_int), ("device", C.c_int)]


class TpDem(C.Structure):
    _fields_ = [("ncols", C.c_int), ("nrows", C.c_int), ("xll", C.c_double), ("yll", C.c_double),
                ("cellsize", C.c_double), ("z", C.POINTER(C.c_double))]


# every symbol include/tpflow_b200.h declares, with its ctypes signature
_vp, _dp, _ip, _lp = C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_long)
SIGNATURES = {
    "tp_create": (C.c_int, [C.POINTER(TpParams), C.POINTER(TpDem), C.POINTER(_vp)]),
    "tp_create_slab": (C.c_int, [C.POINTER(TpParams), C.POINTER(TpDem), C.c_int, C.c_int, C.POINTER(_vp)]),
    "tp_destroy": (None, [_vp]),
    "tp_last_error": (C.c_char_p, [_vp]),
    "tp_geometry": (C.c_int, [C.POINTER(TpDem), C.c_double, _dp]),
    "tp_dims": (C.c_int, [_vp, _ip, _ip, _dp, _dp]),
    "tp_set_option": (C.c_int, [_vp, C.c_char_p, C.c_long]),
    "tp_set_initial_thickness": (C.c_int, [_vp, _dp]),
    "tp_set_initial_velocity": (C.c_int, [_vp, _dp, _dp]),
    "tp_set_hydrograph": (C.c_int, [_vp, C.c_int, _ip, _ip, C.c_char_p, C.c_int, _dp, _dp, _dp, _dp]),
    "tp_get_state": (C.c_int, [_vp, _dp]),
    "tp_set_state": (C.c_int, [_vp, _dp]),
    "tp_get_geometry": (C.c_int, [_vp, _dp]),
    "tp_apply_boundaries": (C.c_int, [_vp, C.c_double]),
    "tp_compute_dt": (C.c_int, [_vp, C.c_double, C.c_double, _dp]),
    "tp_advance_step": (C.c_int, [_vp, C.c_double, C.c_double]),
    "tp_regularize": (C.c_int, [_vp]),
    "tp_set_advection_only": (C.c_int, [_vp, C.c_int]),
    "tp_steps": (C.c_int, [_vp, C.c_double, C.c_double, C.c_long, _dp, _lp, _ip, _dp]),
    "tp_get_audit": (C.c_int, [_vp, _dp]),
    "tp_set_audit": (C.c_int, [_vp, _dp]),
    "tp_interior_mass": (C.c_int, [_vp, _dp, _dp]),
    "tp_snapshot": (C.c_int, [_vp, _dp]),
    "tp_interior_mass_device": (C.c_int, [_vp, _dp, _dp]),
    "tp_halo_bytes": (C.c_long, [_vp]),
    "tp_halo_pack": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "tp_halo_unpack": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "tp_step_begin": (C.c_int, [_vp, C.c_double, C.c_double, C.c_double]),
    "tp_bc": (C.c_int, [_vp, C.c_int]),
    "tp_lambda_local": (C.c_int, [_vp, _vp]),
    "tp_dt_from": (C.c_int, [_vp, _vp]),
    "tp_stage": (C.c_int, [_vp, C.c_int]),
    "tp_stage_timed": (C.c_int, [_vp, C.c_int, C.POINTER(C.c_float)]),
    "tp_steps_timed": (C.c_int, [_vp, C.c_double, C.c_double, C.c_long, _dp, _lp, _ip, C.POINTER(C.c_float),
                                 C.POINTER(C.c_float)]),
    "tp_step_end": (C.c_int, [_vp, _dp, _ip, _dp]),
    "tp_set_stream": (C.c_int, [_vp, _vp]),
    "tp_synchronize": (C.c_int, [_vp]),
    "tp_device_state": (C.c_int, [_vp, C.c_int, C.POINTER(_vp), _lp, _lp]),
    "tp_kernel_launches": (C.c_long, [_vp]),
    "tp_selftest_division": (C.c_int, [C.c_int, C.c_long, C.c_ulonglong, C.POINTER(C.c_ulonglong)]),
    "tp_selftest_minmod": (C.c_int, [C.c_int, C.c_long, _dp, _dp, _dp]),
    "tp_active_tiles": (C.c_int, [_vp, _ip, _ip, _ip]),
    "tp_timed_tiles": (C.c_int, [_vp, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "tp_peer_export": (C.c_int, [_vp, _vp]),
    "tp_peer_connect": (C.c_int, [_vp, C.c_int, C.c_int, _vp]),
    "tp_peer_connect_local": (C.c_int, [_vp, C.c_int, C.c_int, C.POINTER(_vp)]),
    "tp_steps_group": (C.c_int, [C.POINTER(_vp), C.c_int, C.c_double, C.c_double, C.c_long, _dp, _lp, _ip]),
    "tp_safe_tiles": (C.c_int, [_vp, _ip]),
    "tp_cond_skipped_tiles": (C.c_int, [_vp, C.POINTER(C.c_ulonglong)]),
    "tp_debug_phase_cycles": (C.c_int, [C.POINTER(C.c_ulonglong), C.c_int]),
}


def build(verbose: bool = False) -> str:
    """Compile the CUDA extension in-tree for sm_100a (make -C csrc)."""
    out = subprocess.run(["make", "-C", CSRC], capture_output=True, text=True)
    if out.returncode != 0:
        raise RuntimeError("building libtpflow_b200.so failed:\n" + out.stdout + out.stderr)
    if verbose:
        print(out.stdout)
    return LIB_PATH


_LIB = None


def lib():
    """The loaded C ABI.  Raises (no fallback) when the extension is missing."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(make -C paper_2104_06784_b200/csrc); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            try:
                f = getattr(L, name)
            except AttributeError:
                if "TPFLOW_B200_LIB" in os.environ:  # an older build under test (A/B timing)
                    continue
                raise
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB
