"""Ensemble inputs on the device (the template is reference ``eda.py``).

Builds the BASELINE.json configurations without host
integration: random draws come from the reference's named substreams
(streams.py:16-36; eda.py:87-108 stream names), everything else -- the
2000-step deterministic spin-up, U_B perturbations, the control and member
trajectories, nonlinear observations and innovations -- runs on the GPU
with the bit-exact RK4 producer.
"""

import zlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .assim import Linearization
from .covariance import DiagonalNoise, device_factor, gaussian_factor
from .model import advance_device, integrate_device
from .obs import ObsNetwork, strided_grid


def _key(part):
    if isinstance(part, (int, np.integer)):
        return int(part)
    return zlib.crc32(str(part).encode())


def substream(seed, *path):
    """Named Philox substream (streams.py:16-30)."""
    seq = np.random.SeedSequence(entropy=seed, spawn_key=tuple(_key(p) for p in path))
    return np.random.Generator(np.random.Philox(seq))


@dataclass
class BaselineConfig:
    """One row of SURVEY.md §8.0 (BASELINE.json configs)."""

    name: str
    n: int
    n_steps: int
    obs_stride: int
    obs_every: int
    cov_length: float
    members: int
    shared_linearization: bool
    ell: int
    k: int
    pcg_iters: int
    sketch: str = "rhsdiff"
    forcing: float = 8.0
    dt: float = 0.025
    sigma_obs: float = 1.0
    sigma_bg: float = 0.8
    spinup_steps: int = 2000
    seed: int = 0

    @property
    def obs_times(self):
        return tuple(range(self.obs_every, self.n_steps + 1, self.obs_every))

    @property
    def grid_count(self):
        return self.n // self.obs_stride


BASELINE_CONFIGS = {
    1: BaselineConfig("cfg1", 40, 8, 2, 1, 2.0, 10, True, 10, 10, 30),
    2: BaselineConfig("cfg2", 40, 8, 2, 1, 2.0, 50, False, 50, 50, 50),
    3: BaselineConfig("cfg3", 1024, 16, 4, 2, 8.0, 50, False, 64, 64, 60,
                      sketch="rhsdiff+gaussian"),
    4: BaselineConfig("cfg4", 16384, 24, 4, 3, 16.0, 200, False, 128, 128, 80),
    5: BaselineConfig("cfg5", 262144, 12, 8, 1, 32.0, 256, False, 256, 128, 20),
}


@dataclass
class DeviceEnsemble:
    """Control (row 0) + members (rows 1..M) of one twin experiment."""

    cfg: BaselineConfig
    net: ObsNetwork
    ub: object
    rn: DiagonalNoise
    states: torch.Tensor       # (M+1 or 1+n_own, N+1, n) linearization trajectories
    innovations: torch.Tensor  # (M+1, p)
    traj_of: np.ndarray        # row -> trajectory index
    lin: Linearization = None
    x0: torch.Tensor = None    # (M+1, n) initial states: x_b and the member x_j
    y: torch.Tensor = None     # (M+1, p) (perturbed) observations y, y_j
    grid_t: torch.Tensor = None
    times_t: torch.Tensor = None

    @property
    def members(self):
        return self.innovations.shape[0] - 1

    def refresh(self, x0=None, y=None):
        """New assimilation cycle from initial states / observations (host or
        device; copied into the resident buffers): integrate every row on the
        GPU, observe it, innovations d_j = y_j - G(x_j) (eda.py:99-105).  All
        device buffers keep their addresses, so operators built on them stay
        valid."""
        if x0 is not None:
            self.x0.copy_(x0, non_blocking=True)
        if y is not None:
            self.y.copy_(y, non_blocking=True)
        cfg = self.cfg
        n, N = cfg.n, cfg.n_steps
        rows = self.x0.shape[0]
        full = self.states if self.states.shape[0] == rows else self._scratch
        _lib.call("edak_integrate", n, N, float(cfg.dt), float(cfg.forcing), self.x0.data_ptr(), rows,
                  full.data_ptr(), (N + 1) * n, None, 4 * N * n, _lib.stream())
        _lib.call("edak_observe", full.data_ptr(), (N + 1) * n, n, self.grid_t.data_ptr(),
                  self.net.grid.size, self.times_t.data_ptr(), self.net.times.size, rows,
                  self._gx.data_ptr(), _lib.stream())
        torch.sub(self.y, self._gx, out=self.innovations)
        if full is not self.states:
            self.states.copy_(full[: self.states.shape[0]])


def _normal_block(seed, path_fn, rows, size):
    out = np.empty((len(rows), size))
    for i, j in enumerate(rows):
        out[i] = substream(seed, *path_fn(j)).standard_normal(size)
    return out


def build_ensemble(cfg, members=None, member_offset=0, truth=None):
    """Device twin experiment for a BASELINE config.

    members / member_offset select member ids member_offset+1 ..
    member_offset+members (multi-GPU sharding keeps the reference stream ids).
    Returns a DeviceEnsemble whose Linearization holds the control
    trajectory and each member's own (or, shared mode, only the control);
    only the states are kept (the sweeps recompute the RK4 stages)."""
    members = cfg.members if members is None else members
    dev = _dev.device()
    n, N = cfg.n, cfg.n_steps
    net = ObsNetwork(strided_grid(n, cfg.grid_count), cfg.obs_times)
    ub = gaussian_factor(n, cfg.sigma_bg, cfg.cov_length)
    rn = DiagonalNoise(cfg.sigma_obs)
    df = device_factor(ub)
    x_true = (truth if truth is not None
              else advance_device(_truth0(cfg), cfg.dt, cfg.spinup_steps, cfg.forcing)[0])
    x_true = torch.as_tensor(x_true, dtype=torch.float64, device=dev)
    truth_states, _ = integrate_device(x_true[None], cfg.dt, N, cfg.forcing)
    grid_t, times_t = _dev.i32(net.grid), _dev.i32(net.times)
    p = net.p
    y = torch.empty((1, p), dtype=torch.float64, device=dev)
    _lib.call("edak_observe", truth_states.data_ptr(), (N + 1) * n, n, grid_t.data_ptr(),
              net.grid.size, times_t.data_ptr(), net.times.size, 1, y.data_ptr(), _lib.stream())
    y = y + cfg.sigma_obs * _dev.f64(substream(cfg.seed, "obsnoise").standard_normal(p))[None]
    # backgrounds: x_b = x_t + U_B eta_0; x_j = x_b + U_B eta_j (eda.py:93-102)
    ids = list(range(member_offset + 1, member_offset + members + 1))
    eta = _dev.f64(_normal_block(cfg.seed, lambda j: ("bg", j), [0] + ids, n))
    # the control's and the members' perturbations as separate blocks: the
    # overlap-save U_B pairs columns (2c, 2c + 1), so a member's bits depend
    # only on its id, never on the control row (even shards are bit-identical)
    pert = torch.cat([df.apply_cols(eta[:1]), df.apply_cols(eta[1:])], 0)
    x_bg = x_true[None] + pert[:1]
    x0 = torch.cat([x_bg, x_bg + pert[1:]], 0).contiguous()
    states, _ = integrate_device(x0, cfg.dt, N, cfg.forcing)
    # innovations d_j = y_j - G(x_j) against each member's own run (eda.py:103-105)
    gx = torch.empty((members + 1, p), dtype=torch.float64, device=dev)
    _lib.call("edak_observe", states.data_ptr(), (N + 1) * n, n, grid_t.data_ptr(),
              net.grid.size, times_t.data_ptr(), net.times.size, members + 1, gx.data_ptr(),
              _lib.stream())
    eps = _normal_block(cfg.seed, lambda j: ("obsnoise", j), ids, p)
    yj = torch.cat([y, y + cfg.sigma_obs * _dev.f64(eps)], 0)
    innov = (yj - gx).contiguous()
    if cfg.shared_linearization:
        states = states[:1].contiguous()
        traj_of = np.zeros(members + 1, dtype=np.int64)
    else:
        traj_of = np.arange(members + 1)
    ens = DeviceEnsemble(cfg, net, ub, rn, states, innov, traj_of)
    ens.lin = Linearization(states, cfg.dt, cfg.forcing, net, ub, rn)
    ens.x0, ens.y, ens.grid_t, ens.times_t = x0, yj.contiguous(), grid_t, times_t
    ens._gx = gx
    ens._scratch = (None if not cfg.shared_linearization else
                    torch.empty((members + 1, N + 1, n), dtype=torch.float64, device=dev))
    return ens


def _truth0(cfg):
    x = np.full(cfg.n, cfg.forcing, dtype=float)
    x[0] += 0.01
    return x
