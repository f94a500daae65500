"""Shared helpers for the parity tests (test infrastructure)."""
import numpy as np


def bits(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bitwise(got: np.ndarray, want: np.ndarray, what: str = "") -> None:
    g, w = bits(got), bits(want)
    if not np.array_equal(g, w):
        bad = np.argwhere(g != w)
        k = tuple(bad[0])
        raise AssertionError(
            f"{what}: {len(bad)} of {g.size} values differ bitwise; first at {k}: "
            f"got {got[k]!r} want {want[k]!r} (max |diff| {np.nanmax(np.abs(got - want)):.3e})")


def rel_err(got: np.ndarray, want: np.ndarray):
    """relative L1 and Linf error over all entries (north_star gate: <= 1e-9)."""
    d = np.abs(got - want)
    scale1 = max(np.abs(want).sum(), 1e-300)
    scaleinf = max(np.abs(want).max(), 1e-300)
    return d.sum() / scale1, d.max() / scaleinf
