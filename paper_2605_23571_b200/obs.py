"""Observation network (mirrors reference ``obs.py``).

The device kernels address observations through two int32 maps built once
per network: ``gpos[i]`` = position of ring point i in ``grid`` (or -1) and
``tpos[t]`` = position of level t in ``times`` (or -1).  Time-major ordering
(entry t_pos * G + g_pos, obs.py:45,50) therefore holds by construction,
for arbitrary (not only strided) distinct grids and time lists.
"""

from dataclasses import dataclass

import numpy as np
import torch

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

    def observe(self, traj):
        """Nonlinear map (obs.py:43-45): time-major samples of the states."""
        st = getattr(traj, "device_states", None)
        if st is None:  # host trajectory: an integer gather, no arithmetic
            return np.asarray(traj.states)[np.ix_(self.times, self.grid)].ravel()
        from . import _lib
        n, N = st.shape[-1], st.shape[-2] - 1
        dn = DeviceNetwork(self, n, N)
        out = torch.empty((1, self.p), dtype=torch.float64, device=st.device)
        _lib.call("edak_observe", st.data_ptr(), (N + 1) * n, n, dn.grid.data_ptr(), dn.G,
                  dn.times.data_ptr(), dn.T, 1, out.data_ptr(), _lib.stream())
        return out[0].cpu().numpy()

    def _window(self, traj):
        cache = getattr(traj, "_edak_net_lin", None)
        if cache is None:
            cache = {}
            try:
                traj._edak_net_lin = cache
            except AttributeError:
                pass
        lin = cache.get(id(self))
        if lin is None:
            from .assim import Linearization
            from .covariance import CirculantFactor, DiagonalNoise
            st = getattr(traj, "device_states", None)
            st = np.asarray(traj.states) if st is None else st
            n = st.shape[-1]
            lin = Linearization(st, traj.dt, traj.forcing, self,
                                CirculantFactor(n, np.ones(n // 2 + 1)), DiagonalNoise(1.0))
            cache[id(self)] = lin
        return lin

    def observe_tlm(self, traj, v):
        """G'(traj) v (obs.py:47-50): TL sweep with time-major capture."""
        lin = self._window(traj)
        cols, _, as_np = _dev.to_cols(v, lin.n)
        out = lin.tl_cols(cols)[0]
        return out.cpu().numpy() if as_np else out

    def observe_adj(self, traj, w):
        """Adjoint of observe_tlm (obs.py:52-57): AD sweep forced at the
        observed (time, point) pairs."""
        lin = self._window(traj)
        as_np = not isinstance(w, torch.Tensor)
        W = torch.as_tensor(np.asarray(w, dtype=float) if as_np else w,
                            dtype=torch.float64).to(_dev.device()).reshape(1, -1)
        g = lin.ad_cols(W)[0]
        return g.cpu().numpy() if as_np else g


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
