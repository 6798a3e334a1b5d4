"""Per-axis importance grid: containers on the host, transform/refinement on the device.

Mirror of the reference's grid layer (reference: pkg/src/parcube/vegas_grid.py).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .domain import _Frozen, check_dimension

DEFAULT_N_BINS = 500


class VegasGrid(_Frozen):
    """Bin boundaries (d, n_bins+1), pinned to [0,1], strictly increasing (vegas_grid.py:21-43)."""

    __slots__ = ("d", "n_bins", "boundaries")

    def __init__(self, d: int, n_bins: int, boundaries):
        b = np.array(boundaries, dtype=np.float64)
        if b.shape != (d, n_bins + 1):
            raise ValueError(f"boundaries must have shape ({d}, {n_bins + 1})")
        if not np.allclose(b[:, 0], 0.0) or not np.allclose(b[:, -1], 1.0):
            raise ValueError("boundaries must start at 0 and end at 1")
        if np.any(np.diff(b, axis=1) <= 0):
            raise ValueError("boundaries must be strictly increasing")
        b[:, 0], b[:, -1] = 0.0, 1.0
        b.setflags(write=False)
        self._put("d", int(d))
        self._put("n_bins", int(n_bins))
        self._put("boundaries", b)

    def widths(self) -> np.ndarray:
        return np.diff(self.boundaries, axis=1)


class BinContributions:
    """Accumulated squared sample contributions, one row per axis (vegas_grid.py:46-62)."""

    def __init__(self, d: int, n_bins: int):
        self.d = check_dimension(d)
        self.n_bins = int(n_bins)
        self.c = np.zeros((self.d, self.n_bins))

    def reset(self) -> None:
        self.c.fill(0.0)

    def total(self) -> np.ndarray:
        return self.c.sum(axis=1)


class GridRefineParams(_Frozen):
    """Damping exponent and smoothing switch (vegas_grid.py:65-75)."""

    __slots__ = ("alpha", "smoothing")

    def __init__(self, alpha: float = 1.5, smoothing: bool = True):
        if alpha < 0:
            raise ValueError("alpha must be >= 0")
        self._put("alpha", float(alpha))
        self._put("smoothing", bool(smoothing))


def check_grid_shape(d: int, n_bins: int):
    """The argument checks of init_grid (vegas_grid.py:77-84) without building the table: the device-resident run
    starts from its own uniform grid and a (d, 501) host table plus its validation cost ~100 us per call."""
    d = check_dimension(d)
    n_bins = int(n_bins)
    if n_bins < 2:
        raise ValueError("n_bins must be >= 2")
    return d, n_bins


def init_grid(d: int, n_bins: int = DEFAULT_N_BINS) -> VegasGrid:
    """Uniform grid k / n_bins (vegas_grid.py:77-84)."""
    d, n_bins = check_grid_shape(d, n_bins)
    return VegasGrid(d, n_bins, np.tile(np.arange(n_bins + 1) / n_bins, (d, 1)))


def transform_many(y, grid: VegasGrid, device=None):
    """(x, jacobian, bin_ids) for an (n, d) array of uniform points (vegas_grid.py:99-114), on the device."""
    y = np.asarray(y, dtype=float)
    if y.ndim != 2 or y.shape[1] != grid.d:
        raise ValueError(f"expected (n, {grid.d}) points")
    return _native.grid_transform(grid.boundaries, y, device=device)


def transform(y, grid: VegasGrid):
    """One uniform point through the grid (vegas_grid.py:87-96)."""
    y = np.atleast_1d(np.asarray(y, dtype=float))
    x, jac, bins = transform_many(y[None, :], grid)
    return x[0], float(jac[0]), bins[0]


def refine_grid(grid: VegasGrid, contributions: BinContributions, params: GridRefineParams | None = None,
                device=None) -> VegasGrid:
    """Equal-damped-contribution boundaries, per axis (vegas_grid.py:142-193); csrc/mcubes_aux.cuh."""
    params = params or GridRefineParams()
    if contributions.d != grid.d or contributions.n_bins != grid.n_bins:
        raise ValueError("contribution table does not match grid shape")
    new_b = _native.grid_refine(grid.boundaries, contributions.c, params.alpha, params.smoothing, device=device)
    return VegasGrid(grid.d, grid.n_bins, new_b)


def grid_snapshot_text(grid: VegasGrid) -> str:
    """Boundary dump, one line per axis (vegas_grid.py:196-202)."""
    rows = [f"# d={grid.d} n_bins={grid.n_bins}"]
    rows += [f"axis {j}: " + " ".join(f"{v:.12g}" for v in grid.boundaries[j]) for j in range(grid.d)]
    return "\n".join(rows) + "\n"
