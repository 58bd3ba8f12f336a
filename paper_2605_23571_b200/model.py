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


# ---- per-vector operators (model.py:20-84) on the device ------------------
# numpy (n,) in -> numpy out; device tensors (n,) or (ncols, n) -> tensors.
# Every operation is IEEE-rounded in the reference's numpy order, so the
# results equal the reference's bit for bit.

def _vec_in(*arrays):
    host = not isinstance(arrays[0], torch.Tensor)
    out = []
    for a in arrays:
        t = torch.as_tensor(np.asarray(a, dtype=float) if host else a, dtype=torch.float64)
        out.append(t.to(_dev.device()).contiguous())
    return host, out


def _vec_out(host, t):
    return t.cpu().numpy() if host else t


def _dims(t):
    return (t.shape[-1], 1 if t.dim() == 1 else t.shape[0])


def _tend(op, x, v, forcing=0.0):
    out = torch.empty_like(x)
    n, m = _dims(x)
    if op == 0:
        _lib.call("edak_tendency", n, m, x.data_ptr(), float(forcing), out.data_ptr(), _lib.stream())
    else:
        _lib.call("edak_tendency_tlm" if op == 1 else "edak_tendency_adj", n, m, x.data_ptr(),
                  v.data_ptr(), out.data_ptr(), _lib.stream())
    return out


def _axpy(y, c, z):
    """y + c z, or c z for y None."""
    out = torch.empty_like(z)
    _lib.call("edak_axpy_rn", z.numel(), _lib.ptr(y), float(c), z.data_ptr(), out.data_ptr(),
              _lib.stream())
    return out


def _combine(y, c, a1, a2, a3, a4):
    out = torch.empty_like(y)
    _lib.call("edak_rk4_combine", y.numel(), y.data_ptr(), float(c), a1.data_ptr(), a2.data_ptr(),
              a3.data_ptr(), a4.data_ptr(), out.data_ptr(), _lib.stream())
    return out


def tendency(x, forcing):
    """Time derivative of the cyclic Lorenz-96 state (model.py:20-22)."""
    host, (xd,) = _vec_in(x)
    return _vec_out(host, _tend(0, xd, None, forcing))


def tendency_tlm(x, v):
    """J(x) v (model.py:25-28)."""
    host, (xd, vd) = _vec_in(x, v)
    return _vec_out(host, _tend(1, xd, vd))


def tendency_adj(x, w):
    """J(x)^T w (model.py:31-35)."""
    host, (xd, wd) = _vec_in(x, w)
    return _vec_out(host, _tend(2, xd, wd))


def _rk4_stages(x, dt, forcing):
    """One RK4 step: (new state, (x, x2, x3, x4)) (model.py:38-48)."""
    host, (xd,) = _vec_in(x)
    k1 = _tend(0, xd, None, forcing)
    x2 = _axpy(xd, 0.5 * dt, k1)
    k2 = _tend(0, x2, None, forcing)
    x3 = _axpy(xd, 0.5 * dt, k2)
    k3 = _tend(0, x3, None, forcing)
    x4 = _axpy(xd, dt, k3)
    k4 = _tend(0, x4, None, forcing)
    xn = _combine(xd, dt / 6.0, k1, k2, k3, k4)
    return _vec_out(host, xn), tuple(_vec_out(host, t) for t in (xd, x2, x3, x4))


def step_tlm(stages, dt, v):
    """Tangent-linear of one RK4 step around stored stages (model.py:56-63)."""
    host, (x1, x2, x3, x4, vd) = _vec_in(*stages, v)
    a1 = _tend(1, x1, vd)
    a2 = _tend(1, x2, _axpy(vd, 0.5 * dt, a1))
    a3 = _tend(1, x3, _axpy(vd, 0.5 * dt, a2))
    a4 = _tend(1, x4, _axpy(vd, dt, a3))
    return _vec_out(host, _combine(vd, dt / 6.0, a1, a2, a3, a4))


def step_adj(stages, dt, w):
    """Adjoint of step_tlm around the same stages (model.py:66-84)."""
    host, (x1, x2, x3, x4, wd) = _vec_in(*stages, w)
    a4 = _axpy(None, dt / 6.0, wd)
    a3 = _axpy(None, 2.0 * dt / 6.0, wd)
    a2 = _axpy(None, 2.0 * dt / 6.0, wd)
    a1 = _axpy(None, dt / 6.0, wd)
    u4 = _tend(2, x4, a4)
    vhat = _axpy(wd, 1.0, u4)
    a3 = _axpy(a3, dt, u4)
    u3 = _tend(2, x3, a3)
    vhat = _axpy(vhat, 1.0, u3)
    a2 = _axpy(a2, 0.5 * dt, u3)
    u2 = _tend(2, x2, a2)
    vhat = _axpy(vhat, 1.0, u2)
    a1 = _axpy(a1, 0.5 * dt, u2)
    vhat = _axpy(vhat, 1.0, _tend(2, x1, a1))
    return _vec_out(host, vhat)


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


def spinup(n, dt, forcing, n_steps, rng):
    """On-attractor state (model.py:160-166): the rest state plus 1e-3 N(0,1)
    from the host stream, then ``n_steps`` free RK4 steps on the GPU."""
    x = np.full(n, forcing, dtype=float)
    x += 1e-3 * rng.standard_normal(n)
    return advance_device(x, dt, n_steps, forcing)[0].cpu().numpy()


class DeviceTrajectory:
    """Trajectory whose states live on the device (eda.build_setup); the
    reference attributes ``states`` / ``stages`` are host copies made on
    first access (stages recomputed on the GPU, bit-exact)."""

    def __init__(self, device_states, dt, forcing):
        self.device_states = device_states  # (N+1, n) view
        self.dt = float(dt)
        self.forcing = float(forcing)
        self._states = None
        self._stages = None

    @property
    def n_steps(self):
        return self.device_states.shape[0] - 1

    @property
    def n(self):
        return self.device_states.shape[1]

    @property
    def states(self):
        if self._states is None:
            self._states = self.device_states.cpu().numpy()
        return self._states

    @property
    def stages(self):
        if self._stages is None:
            N = self.n_steps
            _, sg = integrate_device(self.device_states[:N], self.dt, 1, self.forcing,
                                     want_stages=True)
            self._stages = sg[:, 0].cpu().numpy()
        return self._stages


def _full_window_operator(traj):
    """Linearization of ``traj`` whose observation network is every grid
    point at every level (0..N) with R = I and U_B = I: its TL sweep returns
    the whole perturbation history, its AD sweep takes a dense forcing."""
    from .assim import Linearization
    from .covariance import CirculantFactor, DiagonalNoise
    from .obs import ObsNetwork
    lin = getattr(traj, "_edak_full_lin", None)
    if lin is None:
        st = getattr(traj, "device_states", None)
        st = np.asarray(traj.states) if st is None else st
        n, N = st.shape[-1], st.shape[-2] - 1
        net = ObsNetwork(np.arange(n), np.arange(N + 1))
        lin = Linearization(st, traj.dt, traj.forcing, net,
                            CirculantFactor(n, np.ones(n // 2 + 1)), DiagonalNoise(1.0))
        try:
            traj._edak_full_lin = lin
        except AttributeError:
            pass
    return lin


def tlm(traj, v0):
    """Tangent-linear sweep (model.py:134-144): all N+1 levels, (N+1, n)."""
    lin = _full_window_operator(traj)
    cols, _, as_np = _dev.to_cols(v0, lin.n)
    out = lin.tl_cols(cols).reshape(lin.n_steps + 1, lin.n)
    return out.cpu().numpy() if as_np else out


def adjoint(traj, w_all):
    """Adjoint sweep (model.py:147-157): g with <tlm(traj, v), w_all> = <v, g>."""
    lin = _full_window_operator(traj)
    as_np = not isinstance(w_all, torch.Tensor)
    W = torch.as_tensor(np.asarray(w_all, dtype=float) if as_np else w_all,
                        dtype=torch.float64).to(_dev.device()).reshape(1, -1)
    g = lin.ad_cols(W)[0]
    return g.cpu().numpy() if as_np else g
