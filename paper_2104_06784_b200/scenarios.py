"""Deterministic synthetic inputs for the BASELINE.json configs.

The reference only *declares* its scenario generators
(/root/reference/proj/include/tpflow/scenarios.hpp:12-33, no definitions anywhere),
so this module supplies them.  Everything is plain float64 numpy evaluated once on
the host; the same arrays are fed to the CUDA path and to the CPU oracle, so
parity never depends on these formulas being reproduced elsewhere.

Conventions follow the reference DEM (terrain.hpp:12-14): arrays are
``[nrows, ncols]`` with row j=0 the SOUTH row, column i=0 the WEST column,
elevations in metres.  A scenario is a :class:`Scenario` bundle of DEM, the
Mode-I thickness/velocity grids or the Mode-II hydrograph, and the config.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Optional

import numpy as np

from .config import SimConfig, Hydrograph


@dataclasses.dataclass
class Scenario:
    name: str
    z: np.ndarray                      # [nrows, ncols] metres, south row first
    cellsize: float
    config: SimConfig
    h0: Optional[np.ndarray] = None    # Mode-I thickness, metres
    vx0: Optional[np.ndarray] = None   # Mode-I velocity, m/s
    vy0: Optional[np.ndarray] = None
    hydrograph: Optional[Hydrograph] = None
    xll: float = 0.0
    yll: float = 0.0

    @property
    def nrows(self) -> int:
        return self.z.shape[0]

    @property
    def ncols(self) -> int:
        return self.z.shape[1]


def _grid(ncols: int, nrows: int, cellsize: float):
    x = (np.arange(ncols, dtype=np.float64) + 0.5) * cellsize
    y = (np.arange(nrows, dtype=np.float64) + 0.5) * cellsize
    return np.meshgrid(x, y)  # X, Y each [nrows, ncols]


# --- DEMs (scenarios.hpp:15-27) -------------------------------------------

def flat_dem(ncols, nrows, cellsize, z0=0.0):
    return np.full((nrows, ncols), float(z0))


def incline_dem(ncols, nrows, cellsize, slope_deg):
    """Plane descending in -X at ``slope_deg`` (scenarios.hpp:18)."""
    X, _ = _grid(ncols, nrows, cellsize)
    return X * math.tan(math.radians(slope_deg))


def bowl_dem(ncols, nrows, cellsize, depth):
    """Closed paraboloid basin z = depth (r/R)^2 centred, transpose-symmetric (scenarios.hpp:20-22)."""
    X, Y = _grid(ncols, nrows, cellsize)
    cx, cy = ncols * cellsize / 2.0, nrows * cellsize / 2.0
    R = min(cx, cy)
    return depth * (((X - cx) ** 2 + (Y - cy) ** 2) / (R * R))


def channel_dem(ncols, nrows, cellsize, slope_deg, wall_height):
    """Straight channel descending in -X with parabolic side walls (scenarios.hpp:24-26)."""
    X, Y = _grid(ncols, nrows, cellsize)
    cy = nrows * cellsize / 2.0
    half = nrows * cellsize / 2.0
    return X * math.tan(math.radians(slope_deg)) + wall_height * ((Y - cy) / half) ** 2


def hill_incline_dem(ncols, nrows, cellsize, slope_deg, hill_h, hill_sigma_frac, hill_cx_frac=0.45):
    """C1: plane tilted down-slope (-X) plus a Gaussian hill."""
    X, Y = _grid(ncols, nrows, cellsize)
    W, H = ncols * cellsize, nrows * cellsize
    s = hill_sigma_frac * W
    hill = hill_h * np.exp(-(((X - hill_cx_frac * W) ** 2 + (Y - 0.5 * H) ** 2) / (2.0 * s * s)))
    return X * math.tan(math.radians(slope_deg)) + hill


def valley_dem(ncols, nrows, cellsize, slope_deg=8.0, wall=400.0, ripple=2.0):
    """C2: parabolic valley descending in -X plus a low-amplitude sinusoid."""
    X, Y = _grid(ncols, nrows, cellsize)
    W, H = ncols * cellsize, nrows * cellsize
    v = ((Y - 0.5 * H) / (0.5 * H)) ** 2
    rip = ripple * np.sin(2 * math.pi * X / (W / 7.0)) * np.cos(2 * math.pi * Y / (H / 5.0))
    return X * math.tan(math.radians(slope_deg)) + wall * v + rip


def fractal_dem(ncols, nrows, cellsize, seed=2104, n_modes=24, relief=300.0, slope_deg=6.0):
    """C4/C5: seeded sum of sinusoids (seed 2104)."""
    rng = np.random.default_rng(seed)
    X, Y = _grid(ncols, nrows, cellsize)
    W, H = ncols * cellsize, nrows * cellsize
    z = X * math.tan(math.radians(slope_deg))
    for k in range(n_modes):
        kx = rng.integers(1, 9)
        ky = rng.integers(1, 9)
        amp = relief / (1.0 + (kx * kx + ky * ky) ** 0.75)
        ph = rng.uniform(0, 2 * math.pi, size=2)
        z = z + amp * np.sin(2 * math.pi * kx * X / W + ph[0]) * np.sin(2 * math.pi * ky * Y / H + ph[1])
    return z


# --- Releases and hydrographs (scenarios.hpp:28-33) -------------------------

def gaussian_release(ncols, nrows, amplitude, width, cx, cy, base=0.0):
    """h = amplitude exp(-r^2/width^2) + base, centre/width in cell units (scenarios.hpp:28-30)."""
    jj, ii = np.meshgrid(np.arange(nrows, dtype=np.float64), np.arange(ncols, dtype=np.float64),
                         indexing="ij")
    r2 = (ii - cx) ** 2 + (jj - cy) ** 2
    return amplitude * np.exp(-r2 / (width * width)) + base


def paraboloid_release(ncols, nrows, h0, rx, ry, cx, cy):
    """Compact release h = h0 max(0, 1 - (dx/rx)^2 - (dy/ry)^2), true dry cells outside (cell units)."""
    jj, ii = np.meshgrid(np.arange(nrows, dtype=np.float64), np.arange(ncols, dtype=np.float64),
                         indexing="ij")
    return h0 * np.maximum(0.0, 1.0 - ((ii - cx) / rx) ** 2 - ((jj - cy) / ry) ** 2)


def triangular_hydrograph(ncols, nrows, side, first_cell, n_cells, t0, t1, peak_h, phi_s, peak_speed):
    """Zero at t0, peak at (t0+t1)/2, zero at t1 (scenarios.hpp:31-33)."""
    cells = []
    for k in range(first_cell, first_cell + n_cells):
        if side == "E":
            cells.append((ncols - 1, k, "E"))
        elif side == "W":
            cells.append((0, k, "W"))
        elif side == "N":
            cells.append((k, nrows - 1, "N"))
        elif side == "S":
            cells.append((k, 0, "S"))
        else:
            raise ValueError(side)
    tm = 0.5 * (t0 + t1)
    samples = [(t0, 0.0, phi_s, 0.0), (tm, peak_h, phi_s, peak_speed), (t1, 0.0, phi_s, 0.0)]
    return Hydrograph(cells=cells, samples=samples)


# --- The BASELINE.json configs ----------------------------------------------

def c1_hill(n=256, t_end=1.0e4, dt_out=1.0e4) -> Scenario:
    """configs[0]: two-phase release on an inclined plane with a Gaussian hill, 256^2, Δ=5 m."""
    cs = 5.0
    z = hill_incline_dem(n, n, cs, slope_deg=15.0, hill_h=20.0, hill_sigma_frac=0.1)
    h0 = paraboloid_release(n, n, h0=5.0, rx=0.12 * n, ry=0.12 * n, cx=0.72 * n, cy=0.5 * n)
    cfg = SimConfig(mode="release", t_end=t_end, dt_out=dt_out)
    return Scenario("C1-hill", z, cs, cfg, h0=h0)


def c2_valley(ncols=2048, nrows=2048, t_end=1.0e4, dt_out=1.0e4) -> Scenario:
    """configs[1]: Mode-I release on a synthetic valley, 2048^2, Δ=5 m.

    The release is a wide compact paraboloid on the valley floor (≈38 % of the
    cells wet at t=0, true dry cells elsewhere)."""
    cs = 5.0
    z = valley_dem(ncols, nrows, cs)
    h0 = paraboloid_release(ncols, nrows, h0=8.0, rx=0.35 * ncols, ry=0.35 * nrows,
                            cx=0.55 * ncols, cy=0.5 * nrows)
    cfg = SimConfig(mode="release", t_end=t_end, dt_out=dt_out)
    return Scenario("C2-valley", z, cs, cfg, h0=h0)


def c3_channel(ncols=4096, nrows=2048, t_end=120.0, dt_out=0.5) -> Scenario:
    """configs[2]: Mode-II inflow on a channel; dry bed, hydrograph starts at h=0."""
    cs = 5.0
    z = channel_dem(ncols, nrows, cs, slope_deg=10.0, wall_height=60.0)
    nin = max(4, nrows // 8)
    hg = triangular_hydrograph(ncols, nrows, "E", nrows // 2 - nin // 2, nin, 0.0, 120.0,
                               peak_h=4.0, phi_s=0.55, peak_speed=5.0)
    cfg = SimConfig(mode="inflow", t_end=t_end, dt_out=dt_out)
    return Scenario("C3-channel", z, cs, cfg, hydrograph=hg)


def c4_terrain(ncols=6000, nrows=4000, t_end=1.0e4, dt_out=1.0e4, seed=2104) -> Scenario:
    """configs[3]: Hsiaolin-scale synthetic terrain, seeded, several compact releases."""
    cs = 5.0
    z = fractal_dem(ncols, nrows, cs, seed=seed)
    rng = np.random.default_rng(seed + 1)
    h0 = np.zeros((nrows, ncols))
    for _ in range(6):
        cx, cy = rng.uniform(0.15, 0.85) * ncols, rng.uniform(0.15, 0.85) * nrows
        r = rng.uniform(0.05, 0.12) * min(ncols, nrows)
        h0 = h0 + paraboloid_release(ncols, nrows, h0=rng.uniform(4, 12), rx=r, ry=r, cx=cx, cy=cy)
    cfg = SimConfig(mode="release", t_end=t_end, dt_out=dt_out)
    return Scenario("C4-terrain", z, cs, cfg, h0=h0)


def wet_valley(ncols, nrows, t_end=1.0e4, dt_out=1.0e4) -> Scenario:
    """Fully wet variant of C2 (every interior cell wet): the worst-case compute load per cell."""
    s = c2_valley(ncols, nrows, t_end, dt_out)
    s.h0 = s.h0 + 0.5
    s.name = "C2-valley-wet"
    return s


def stacked(sc: Scenario, copies: int) -> Scenario:
    """`copies` copies of a Mode-I scenario stacked along the rows (weak scaling: one copy per
    row slab, so every GPU carries the single-GPU workload; the copies couple through the
    shared rows at the seams).  Mode-II hydrographs are not stacked."""
    if sc.hydrograph is not None:
        raise ValueError("stacked: Mode-II scenarios are not supported")
    tile = lambda a: None if a is None else np.ascontiguousarray(np.tile(a, (copies, 1)))  # noqa: E731
    return Scenario(f"{sc.name}x{copies}", tile(sc.z), sc.cellsize, sc.config, h0=tile(sc.h0),
                    vx0=tile(sc.vx0), vy0=tile(sc.vy0), xll=sc.xll, yll=sc.yll)


def moving_release(ncols, nrows, t_end=1.0e4, dt_out=1.0e4, seed=7) -> Scenario:
    """Mode-I release with an initial velocity field (set_initial_velocity, solver.cpp:57-81):
    the C4 terrain with a swirling, noisy velocity everywhere (zero-thickness cells included)."""
    sc = c4_terrain(ncols, nrows, t_end=t_end, dt_out=dt_out, seed=2104 + seed)
    rng = np.random.default_rng(seed)
    y, x = np.mgrid[0:nrows, 0:ncols].astype(np.float64)
    cx, cy = 0.5 * ncols, 0.5 * nrows
    sc.vx0 = -3.0 * (y - cy) / max(nrows, 1) + rng.normal(0.0, 0.5, (nrows, ncols))
    sc.vy0 = 3.0 * (x - cx) / max(ncols, 1) + rng.normal(0.0, 0.5, (nrows, ncols))
    sc.name = "moving-release"
    return sc


def four_side_inflow(ncols, nrows, t_end=30.0, dt_out=0.5) -> Scenario:
    """Mode-II inflow through all four sides (solver.cpp:108-136: per-side ghost rows and
    inward velocity), both cells of the SE corner listed on two sides, a hydrograph that
    starts wet at t=0 and ends (zero after the last sample) before t_end."""
    cs = 5.0
    z = bowl_dem(ncols, nrows, cs, depth=30.0)
    cells = [(0, j, "W") for j in range(nrows // 4, nrows // 4 + 6)]
    cells += [(i, nrows - 1, "N") for i in range(ncols // 3, ncols // 3 + 7)]
    cells += [(i, 0, "S") for i in range(ncols - 5, ncols)]
    cells += [(ncols - 1, j, "E") for j in range(0, 4)]
    samples = [(0.0, 0.5, 0.6, 1.0), (8.0, 3.0, 0.45, 4.0), (20.0, 0.0, 0.5, 0.0)]
    cfg = SimConfig(mode="inflow", t_end=t_end, dt_out=dt_out)
    return Scenario("four-side-inflow", z, cs, cfg, hydrograph=Hydrograph(cells=cells, samples=samples))


SCENARIOS = {
    "c1": c1_hill,
    "c2": c2_valley,
    "c3": c3_channel,
    "c4": c4_terrain,
    "wet": wet_valley,
    "moving": moving_release,
    "inflow4": four_side_inflow,
}
