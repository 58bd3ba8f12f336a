"""Lorenz-96 linearization trajectories (mirrors reference ``model.py``).

``Trajectory`` is the reference container (model.py:87-115).  ``integrate``
keeps the reference signature (model.py:118-131) but runs the sm_100a RK4
producer (``edak_integrate``), bit-exact with the reference because every
stage is evaluated with IEEE-rounded operations in the reference's order.
``integrate_device`` is the batched, device-resident form the ensemble
engine uses (no host round trip).
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib


@dataclass
class Trajectory:
    """states (N+1, n), stages (N, 4, n), dt, forcing (model.py:87-115)."""

    states: np.ndarray
    stages: np.ndarray
    dt: float
    forcing: float

    @property
    def n_steps(self):
        return self.states.shape[0] - 1

    @property
    def n(self):
        return self.states.shape[1]


def integrate_device(x0, dt, n_steps, forcing, want_stages=False):
    """Batched nonlinear runs on the GPU.

    x0: (ncols, n) device tensor (or numpy).  Returns states (ncols, N+1, n)
    and, if requested, stages (ncols, N, 4, n), both device tensors."""
    x0 = torch.as_tensor(x0, dtype=torch.float64, device=_dev.device())
    if x0.dim() == 1:
        x0 = x0[None]
    x0 = x0.contiguous()
    m, n = x0.shape
    states = torch.empty((m, n_steps + 1, n), dtype=torch.float64, device=x0.device)
    stages = (torch.empty((m, n_steps, 4, n), dtype=torch.float64, device=x0.device)
              if want_stages else None)
    _lib.call("edak_integrate", n, n_steps, float(dt), float(forcing), x0.data_ptr(), m,
              states.data_ptr(), (n_steps + 1) * n, _lib.ptr(stages), 4 * n_steps * n,
              _lib.stream())
    return states, stages


def integrate(x0, dt, n_steps, forcing):
    """Reference-signature integrate (model.py:118-131) on the GPU."""
    states, stages = integrate_device(np.asarray(x0, dtype=float)[None], dt, n_steps,
                                      forcing, want_stages=True)
    return Trajectory(states[0].cpu().numpy(), stages[0].cpu().numpy(), dt, forcing)


def rk4_step(x, dt, forcing):
    """One RK4 step (model.py:51-53) on the GPU."""
    states, _ = integrate_device(np.asarray(x, dtype=float)[None], dt, 1, forcing)
    return states[0, 1].cpu().numpy()


def advance_device(x, dt, n_steps, forcing, chunk=64):
    """x after ``n_steps`` RK4 steps (spin-up) for a (ncols, n) device block,
    without keeping the intermediate levels."""
    x = torch.as_tensor(x, dtype=torch.float64, device=_dev.device())
    if x.dim() == 1:
        x = x[None]
    done = 0
    while done < n_steps:
        k = min(chunk, n_steps - done)
        states, _ = integrate_device(x, dt, k, forcing)
        x = states[:, -1].contiguous()
        done += k
    return x


def deterministic_truth(n, dt, forcing, n_steps, bump=0.01):
    """BASELINE truth: x = F, x_0 += bump, ``n_steps`` RK4 steps (device)."""
    x = np.full(n, forcing, dtype=float)
    x[0] += bump
    return advance_device(x, dt, n_steps, forcing)[0]
