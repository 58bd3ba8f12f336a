"""Observation network (mirrors reference ``obs.py``).

The device kernels address observations through two int32 maps built once
per network: ``gpos[i]`` = position of ring point i in ``grid`` (or -1) and
``tpos[t]`` = position of level t in ``times`` (or -1).  Time-major ordering
(entry t_pos * G + g_pos, obs.py:45,50) therefore holds by construction,
for arbitrary (not only strided) distinct grids and time lists.
"""

from dataclasses import dataclass

import numpy as np

from . import _dev


def strided_grid(n, n_observed):
    """obs.py:17-20."""
    return np.arange(n_observed) * (n // n_observed)


@dataclass
class ObsNetwork:
    """Observed grid indices x observed time levels (obs.py:23-41)."""

    grid: np.ndarray
    times: np.ndarray

    def __post_init__(self):
        self.grid = np.asarray(self.grid, dtype=int)
        self.times = np.asarray(self.times, dtype=int)
        if np.unique(self.grid).size != self.grid.size:
            raise ValueError("observed grid points must be distinct")
        if np.unique(self.times).size != self.times.size:
            raise ValueError("observed time levels must be distinct")

    @property
    def p(self):
        return self.grid.size * self.times.size


def position_maps(net, n, n_steps):
    """(gpos[n], tpos[N+1]) int32 host arrays for any ObsNetwork duck type."""
    grid = np.asarray(net.grid, dtype=np.int64)
    times = np.asarray(net.times, dtype=np.int64)
    if grid.size and (grid.min() < 0 or grid.max() >= n):
        raise ValueError("observed grid point outside the ring")
    if times.size and (times.min() < 0 or times.max() > n_steps):
        raise ValueError("observed time level outside the window")
    gpos = np.full(n, -1, dtype=np.int32)
    gpos[grid] = np.arange(grid.size, dtype=np.int32)
    tpos = np.full(n_steps + 1, -1, dtype=np.int32)
    tpos[times] = np.arange(times.size, dtype=np.int32)
    return gpos, tpos


class DeviceNetwork:
    """Device copies of the position maps plus the grid/time index lists."""

    def __init__(self, net, n, n_steps):
        gpos, tpos = position_maps(net, n, n_steps)
        self.G = int(np.asarray(net.grid).size)
        self.T = int(np.asarray(net.times).size)
        self.p = self.G * self.T
        self.gpos = _dev.i32(gpos)
        self.tpos = _dev.i32(tpos)
        self.grid = _dev.i32(np.asarray(net.grid))
        self.times = _dev.i32(np.asarray(net.times))
