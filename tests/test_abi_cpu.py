"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/tpflow_b200.h declares, fails loudly without a GPU, and its host
geometry is bit-identical to the reference's (no device needed)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2104_06784_b200 import _lib, scenarios
from tests.util import assert_bitwise

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "tpflow_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tp_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 35
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes binding covers all of them
    assert set(syms) <= set(_lib.SIGNATURES)


def test_sm100a_code_only():
    out = os.popen(f"cuobjdump -lelf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2104_06784_b200.simulator import Simulator, CudaError
    with pytest.raises(CudaError):
        Simulator.from_scenario(scenarios.c1_hill(16))


@pytest.mark.parametrize("make", [lambda: scenarios.c1_hill(50), lambda: scenarios.c4_terrain(70, 44),
                                  lambda: scenarios.channel_dem and scenarios.c3_channel(80, 40)])
def test_host_geometry_bitwise_vs_oracle(make, oracle_kind):
    from oracle.oracle import OracleSim
    sc = make()
    z = np.ascontiguousarray(sc.z)
    dem = _lib.TpDem(sc.ncols, sc.nrows, 0.0, 0.0, sc.cellsize, z.ctypes.data_as(C.POINTER(C.c_double)))
    out = np.empty((14, sc.nrows + 6, sc.ncols + 6))
    assert _lib.lib().tp_geometry(C.byref(dem), sc.config.scaling.L,
                                  out.ctypes.data_as(C.POINTER(C.c_double))) == 0
    assert_bitwise(out, OracleSim(sc, oracle_kind).geometry(), "tp_geometry vs oracle")


def test_config_validation_messages():
    from paper_2104_06784_b200.config import SimConfig, ConfigError, ModelParams
    with pytest.raises(ConfigError, match="cfl must be in"):
        SimConfig(t_end=1, dt_out=1, cfl=0.2).validate()
    with pytest.raises(ConfigError, match="alpha_rho"):
        SimConfig(params=ModelParams(alpha_rho=0.0), t_end=1, dt_out=1).validate()


def test_hydrograph_at_semantics():
    """Hydrograph::at — clamp before, linear inside, ZERO after the last sample
    (hydrograph.hpp:31-45)."""
    from paper_2104_06784_b200.config import Hydrograph
    hg = Hydrograph(cells=[(9, 3, "E")], samples=[(0.0, 0.0, 0.5, 0.0), (60.0, 2.0, 0.5, 1.0)])
    assert hg.at(30.0)[1] == 1.0
    assert hg.at(120.0)[1] == 0.0
    assert hg.at(-1.0) == hg.samples[0]
