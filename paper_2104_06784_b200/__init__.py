"""paper_2104_06784_b200 — B200-native time-stepping core of MoSES_2PDF (arXiv 2104.06784).

The two-phase (solid + fluid) depth-integrated shallow-flow solver of the
reference (`tpflow::Simulator`, /root/reference/proj) re-built as hand-written
sm_100a FP64 kernels behind a C ABI (include/tpflow_b200.h).  Python here is
host plumbing only: configuration types, synthetic scenarios, the ctypes
binding and the reference-shaped `Simulator` front end.
"""
from .config import (ConfigError, Hydrograph, IoError, MassAudit, ModelParams, NumericsError,
                     RunReport, ScalingConfig, SimConfig, TpflowError)

__all__ = ["ConfigError", "Hydrograph", "IoError", "MassAudit", "ModelParams", "NumericsError",
           "RunReport", "ScalingConfig", "SimConfig", "TpflowError", "Simulator", "build"]


def build(verbose: bool = False) -> str:
    from . import _lib
    return _lib.build(verbose)


def __getattr__(name):
    if name == "Simulator":
        from .simulator import Simulator
        return Simulator
    raise AttributeError(name)
