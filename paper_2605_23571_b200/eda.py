"""Identical-twin ensembles on the device (mirrors reference ``eda.py``).

``TwinConfig`` / ``EnsembleSetup`` / ``build_setup`` keep the reference names,
fields, defaults and random streams (eda.py:31-108): the base seed fixes the
spin-up, truth, observation noise and control background; ``trial_seed``
drives the member perturbations; ``shared_linearization`` linearizes every
member around the control trajectory.

Everything numerical runs on the GPU: the 1000-step spin-up, the truth and
the batched control + member runs (bit-exact RK4 producer), the nonlinear
observations, the U_B perturbations (circulant kernel instead of numpy's
FFT: equal to rounding) and the innovations.  All trajectories stay in ONE
device ``Linearization``; ``control`` and ``members`` are views on it
(``MemberProblem.view``) with the reference duck type, and ``ensemble``
batches all members for ``krylov.pcg_members``.
"""

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .assim import Ensemble, Linearization, MemberProblem
from .covariance import DiagonalNoise, GridCovFactor, device_factor
from .model import DeviceTrajectory, integrate_device, spinup
from .obs import DeviceNetwork, ObsNetwork, strided_grid
from .twin import substream


@dataclass
class TwinConfig:
    """eda.py:31-52 (same fields and defaults)."""

    n: int = 1500
    dt: float = 0.025
    n_steps: int = 10
    forcing: float = 8.0
    spinup_steps: int = 1000
    obs_grid_count: int = 50
    obs_times: tuple = (3, 6, 9)
    sigma_obs: float = 0.05
    sigma_bg: float = 0.8
    cov_length: float = 6.0
    cov_passes: int = 10
    members: int = 20
    seed: int = 1234

    @property
    def p(self):
        return self.obs_grid_count * len(self.obs_times)


@dataclass
class EnsembleSetup:
    """eda.py:55-67, plus the device objects the batched solvers take."""

    cfg: TwinConfig
    net: ObsNetwork
    ub: GridCovFactor
    rn: DiagonalNoise
    truth: DeviceTrajectory
    y: np.ndarray
    control: MemberProblem
    members: list = field(default_factory=list)
    lin: Linearization = None
    ensemble: Ensemble = None


def build_setup(cfg, trial_seed=None, shared_linearization=False):
    """Truth, control and members of a twin experiment (eda.py:70-108)."""
    if trial_seed is None:
        trial_seed = cfg.seed
    dev = _dev.device()
    n, N, L = cfg.n, cfg.n_steps, cfg.members
    net = ObsNetwork(strided_grid(n, cfg.obs_grid_count), cfg.obs_times)
    ub = GridCovFactor(n, cfg.sigma_bg, cfg.cov_length, cfg.cov_passes)
    rn = DiagonalNoise(cfg.sigma_obs)
    df = device_factor(ub)
    dn = DeviceNetwork(net, n, N)

    x_true = spinup(n, cfg.dt, cfg.forcing, cfg.spinup_steps, substream(cfg.seed, "spinup"))
    truth_states, _ = integrate_device(x_true[None], cfg.dt, N, cfg.forcing)
    truth = DeviceTrajectory(truth_states[0], cfg.dt, cfg.forcing)

    def observe(states, rows):
        out = torch.empty((rows, net.p), dtype=torch.float64, device=dev)
        _lib.call("edak_observe", states.data_ptr(), (N + 1) * n, n, dn.grid.data_ptr(), dn.G,
                  dn.times.data_ptr(), dn.T, rows, out.data_ptr(), _lib.stream())
        return out

    y = observe(truth_states, 1)[0] + rn.apply(
        _dev.f64(substream(cfg.seed, "obsnoise").standard_normal(net.p)))
    # x_b = x_t + U_b eta_0 ; x_j = x_b + U_b eta_j (eda.py:93-102)
    eta = np.empty((L + 1, n))
    eta[0] = substream(cfg.seed, "bg", 0).standard_normal(n)
    for j in range(1, L + 1):
        eta[j] = substream(trial_seed, "bg", j).standard_normal(n)
    pert = df.apply_cols(_dev.f64(eta))
    x_bg = _dev.f64(x_true)[None] + pert[:1]
    x0 = torch.cat([x_bg, x_bg + pert[1:]], 0).contiguous()
    states, _ = integrate_device(x0, cfg.dt, N, cfg.forcing)
    gx = observe(states, L + 1)
    yj = y[None].repeat(L + 1, 1)
    if L:
        eps = np.stack([substream(trial_seed, "obsnoise", j).standard_normal(net.p)
                        for j in range(1, L + 1)])
        yj[1:] += rn.apply(_dev.f64(eps))
    innov = (yj - gx).contiguous()

    keep = states[:1] if shared_linearization else states
    lin = Linearization(keep.contiguous(), cfg.dt, cfg.forcing, net, ub, rn)
    trajs = [DeviceTrajectory(lin.states[i], cfg.dt, cfg.forcing) for i in range(lin.M)]
    control = MemberProblem.view(lin, 0, innov[0], trajs[0])
    members = []
    for j in range(1, L + 1):
        t = 0 if shared_linearization else j
        members.append(MemberProblem.view(lin, t, innov[j], trajs[t]))
    ens = Ensemble(lin, innov[1:], [m._index for m in members]) if L else None
    return EnsembleSetup(cfg, net, ub, rn, truth, y.cpu().numpy(), control, members, lin, ens)
