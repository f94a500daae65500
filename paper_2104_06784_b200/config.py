"""Host-side configuration types mirroring the reference.

ModelParams      <- /root/reference/proj/include/tpflow/params.hpp:29-51
ScalingConfig    <- params.hpp:12-26
SimConfig        <- config.hpp:12-46
MassAudit        <- config.hpp:60-75
RunReport        <- config.hpp:77-82
Hydrograph       <- hydrograph.hpp:12-77
ConfigError/IoError/NumericsError <- errors.hpp:8-21 (CLI exit codes 2/3/4)

Validation messages are the reference's, so error behaviour is identical.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Tuple


class TpflowError(RuntimeError):
    exit_code = 1


class ConfigError(TpflowError):
    exit_code = 2


class IoError(TpflowError):
    exit_code = 3


class NumericsError(TpflowError):
    exit_code = 4


ERRORS_BY_CODE = {2: ConfigError, 3: IoError, 4: NumericsError}


@dataclasses.dataclass
class ModelParams:
    delta_b: float = 16.0
    C_d: float = 6.0
    N_R: float = 268.0
    theta_b: float = 5.0
    phi_s0: float = 0.5
    alpha_rho: float = 0.4
    chi: float = 1.0

    def tan_delta_b(self) -> float:
        # params.hpp:38 — std::tan(delta_b * M_PI / 180.0); Python's math.tan is the same libm call.
        return math.tan(self.delta_b * math.pi / 180.0)

    def validate(self) -> None:
        if not (0.0 <= self.delta_b < 90.0):
            raise ConfigError("params: delta_b must be in [0, 90) degrees")
        if not (self.C_d >= 0.0):
            raise ConfigError("params: C_d must be >= 0")
        if not (self.N_R > 0.0):
            raise ConfigError("params: N_R must be > 0")
        if not (self.theta_b >= 0.0):
            raise ConfigError("params: theta_b must be >= 0")
        if not (0.0 <= self.phi_s0 <= 1.0):
            raise ConfigError("params: phi_s0 must be in [0, 1]")
        if not (0.0 < self.alpha_rho <= 1.0):
            raise ConfigError("params: alpha_rho must be in (0, 1]")


@dataclasses.dataclass
class ScalingConfig:
    L: float = 1.0
    H: float = 1.0
    g: float = 9.80665

    def epsilon(self) -> float:
        return self.H / self.L

    def t_unit(self) -> float:
        return math.sqrt(self.L / self.g)

    def v_unit(self) -> float:
        return math.sqrt(self.g * self.L)

    def validate(self) -> None:
        if not (self.L > 0.0):
            raise ConfigError("scaling: L must be > 0")
        if not (self.H > 0.0):
            raise ConfigError("scaling: H must be > 0")
        if not (self.g > 0.0):
            raise ConfigError("scaling: g must be > 0")


@dataclasses.dataclass
class SimConfig:
    params: ModelParams = dataclasses.field(default_factory=ModelParams)
    scaling: ScalingConfig = dataclasses.field(default_factory=ScalingConfig)
    mode: str = "release"          # "release" (Mode-I) | "inflow" (Mode-II)
    t_end: float = 0.0
    dt_out: float = 0.0
    cfl: float = 0.1
    h_dry: float = 1e-10
    eps_h: float = 1e-6
    dem_path: str = "<memory>"
    init_path: str = "<memory>"
    hydrograph_path: str = "<memory>"
    out_dir: str = "."

    @property
    def inflow(self) -> bool:
        return self.mode == "inflow"

    def validate(self) -> None:
        # config.hpp:31-45, same order and messages.
        self.params.validate()
        self.scaling.validate()
        if not (0.0 < self.cfl <= 0.125):
            raise ConfigError(f"config: cfl must be in (0, 0.125], got {self.cfl:f}")
        if not (self.t_end > 0.0):
            raise ConfigError("config: t_end must be > 0")
        if not (self.dt_out > 0.0):
            raise ConfigError("config: dt_out must be > 0")
        if not (self.h_dry > 0.0):
            raise ConfigError("config: h_dry must be > 0")
        if not (self.eps_h > 0.0):
            raise ConfigError("config: eps_h must be > 0")
        if not self.dem_path:
            raise ConfigError("config: missing key 'dem'")
        if self.mode == "release" and not self.init_path:
            raise ConfigError("config: missing key 'init' (required in release mode)")
        if self.mode == "inflow" and not self.hydrograph_path:
            raise ConfigError("config: missing key 'hydrograph' (required in inflow mode)")
        if self.mode not in ("release", "inflow"):
            raise ConfigError(f"<memory>: mode must be 'release' or 'inflow', got '{self.mode}'")


@dataclasses.dataclass
class MassAudit:
    initial: float = 0.0
    final_mass: float = 0.0
    injected: float = 0.0
    outflow: float = 0.0
    clipped: float = 0.0

    def drift(self) -> float:
        return self.final_mass - (self.initial + self.injected - self.outflow + self.clipped)

    def reference(self) -> float:
        r = abs(self.initial) + self.injected
        return r if r > 0.0 else 1.0


@dataclasses.dataclass
class RunReport:
    steps: int = 0
    wall_seconds: float = 0.0
    solid: MassAudit = dataclasses.field(default_factory=MassAudit)
    fluid: MassAudit = dataclasses.field(default_factory=MassAudit)


@dataclasses.dataclass
class Hydrograph:
    """cells: (i, j, side) on the interior grid; samples: (t s, h m, phi_s, speed m/s)."""
    cells: List[Tuple[int, int, str]] = dataclasses.field(default_factory=list)
    samples: List[Tuple[float, float, float, float]] = dataclasses.field(default_factory=list)

    def at(self, t: float) -> Tuple[float, float, float, float]:
        """hydrograph.hpp:31-45 — clamped before the first sample, ZERO after the last."""
        s = self.samples
        if not s or t > s[-1][0]:
            return (t, 0.0, 0.0, 0.0)
        if t <= s[0][0]:
            return s[0]
        for k in range(1, len(s)):
            if t <= s[k][0]:
                a, b = s[k - 1], s[k]
                w = (t - a[0]) / (b[0] - a[0])
                return (t, a[1] + w * (b[1] - a[1]), a[2] + w * (b[2] - a[2]), a[3] + w * (b[3] - a[3]))
        return s[-1]

    def validate(self, ncols: int, nrows: int) -> None:
        """hydrograph.hpp:49-77."""
        s = self.samples
        for k in range(1, len(s)):
            if not (s[k][0] > s[k - 1][0]):
                raise ConfigError("hydrograph: sample times must be strictly increasing "
                                  f"(t={s[k][0]:f} after t={s[k - 1][0]:f})")
        for (_, h, phi, speed) in s:
            if h < 0.0:
                raise ConfigError("hydrograph: negative thickness")
            if speed < 0.0:
                raise ConfigError("hydrograph: negative speed")
            if phi < 0.0 or phi > 1.0:
                raise ConfigError("hydrograph: phi_s out of [0, 1]")
        for (i, j, side) in self.cells:
            if side == "N":
                ok = j == nrows - 1
            elif side == "S":
                ok = j == 0
            elif side == "E":
                ok = i == ncols - 1
            elif side == "W":
                ok = i == 0
            else:
                raise ConfigError(f"hydrograph: unknown side '{side}'")
            if i < 0 or i >= ncols or j < 0 or j >= nrows:
                ok = False
            if not ok:
                raise ConfigError(f"hydrograph: cell ({i}, {j}) is not on the boundary ring of side {side}")
