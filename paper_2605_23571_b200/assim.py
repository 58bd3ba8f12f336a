"""Member problems on the GPU (mirrors reference ``assim.py``).

``MemberProblem`` is the drop-in for the reference class of the same name
(assim.py:22-85): same constructor, attributes, methods, matvec ledger and
return types, but every A-application is one batched sm_100a launch
sequence over the whole block (``edak_hessian_block``):

    U_B (circulant taps)  ->  TL sweep + time-major obs capture
    ->  AD sweep with R^-1 forcing  ->  U_B (+ I for hessian_apply)

``Linearization`` is the engine object underneath: device-resident
trajectories of one or many members (with a column -> trajectory map, so a
shared control trajectory and per-member trajectories are the same code
path), the observation position maps and the factor taps.
``Ensemble`` batches many members: all right-hand sides in one launch, one
Hessian column per member per launch (the batched PCG of krylov.py).
"""

import numpy as np
import torch

from . import _dev, _lib
from .covariance import device_factor
from .obs import DeviceNetwork

STAGE_MODES = ("auto", "recompute", "stream")
_MODE_CODE = {"recompute": 0, "stream": 1}


def _prob_struct(n, n_steps, dt, forcing, states, stages, traj_stride, stage_mode,
                 dnet, dfac, sigma2):
    P = _lib.Problem()
    P.n, P.n_steps, P.dt, P.forcing = n, n_steps, float(dt), float(forcing)
    P.states = states.data_ptr() if states is not None else None
    P.stages = stages.data_ptr() if stages is not None else None
    P.traj_stride = traj_stride
    P.stage_mode = _MODE_CODE[stage_mode]
    P.gpos, P.tpos = dnet.gpos.data_ptr(), dnet.tpos.data_ptr()
    P.G, P.T = dnet.G, dnet.T
    P.sigma2 = float(sigma2)
    P.taps, P.ntaps, P.tap_w = dfac.taps.data_ptr(), dfac.ntaps, dfac.tap_w
    P.os_spec, P.os_tw, P.os_logm = _lib.ptr(dfac.os_spec), _lib.ptr(dfac.os_tw), dfac.os_logm
    return P


def stages_recomputable(states, stages, dt, forcing):
    """True iff re-running the RK4 stage chain from ``states[:, s]`` on the
    GPU reproduces ``stages`` bit for bit (then only the states need to be
    kept on the device: 16 instead of 64 bytes per element-step)."""
    m, N, n = states.shape[0], stages.shape[1], states.shape[-1]
    x = states[:, :N].reshape(m * N, n).contiguous()
    st = torch.empty((m * N, 2, n), dtype=torch.float64, device=x.device)
    sg = torch.empty((m * N, 1, 4, n), dtype=torch.float64, device=x.device)
    _lib.call("edak_integrate", n, 1, float(dt), float(forcing), x.data_ptr(), m * N,
              st.data_ptr(), 2 * n, sg.data_ptr(), 4 * n, _lib.stream())
    return bool(torch.equal(sg.reshape(m, N, 4, n), stages))


class Linearization:
    """Device window operator for a set of trajectories sharing (n, N, dt,
    F, network, U_B, R).

    states: (M, N+1, n) or (M, N, n) float64 tensor (device or host).
    stages: optional (M, N, 4, n) -- required for stage_mode "stream",
    used for verification in "auto"."""

    def __init__(self, states, dt, forcing, net, ub, rn, stages=None,
                 stage_mode="recompute"):
        if stage_mode not in STAGE_MODES:
            raise ValueError(f"stage_mode must be one of {STAGE_MODES}")
        dev = _dev.device()
        states = torch.as_tensor(states, dtype=torch.float64).to(dev).contiguous()
        if states.dim() == 2:
            states = states[None]
        self.M, levels, self.n = states.shape
        if stages is not None:
            stages = torch.as_tensor(stages, dtype=torch.float64).to(dev).contiguous()
            if stages.dim() == 3:
                stages = stages[None]
            self.n_steps = stages.shape[1]
        else:
            self.n_steps = levels - 1 if levels > 1 else levels
        if stage_mode == "auto":
            if stages is None:
                stage_mode = "recompute"
            else:
                stage_mode = ("recompute" if stages_recomputable(states, stages, dt, forcing)
                              else "stream")
        if stage_mode == "stream" and stages is None:
            raise ValueError(f"stage_mode={stage_mode!r} needs the stored stages")
        self.stage_mode = stage_mode
        self.states = states
        self.stages = stages if stage_mode == "stream" else None
        self.dt, self.forcing = float(dt), float(forcing)
        self.net, self.ub, self.rn = net, ub, rn
        self.dnet = DeviceNetwork(net, self.n, self.n_steps)
        self.dfac = device_factor(ub)
        self.p = self.dnet.p
        self.sigma2 = float(rn.sigma) ** 2
        stride = (self.stages[0].numel() if self.stages is not None
                  else states[0].numel())
        self._P = _prob_struct(self.n, self.n_steps, dt, forcing, states, self.stages,
                               stride, stage_mode, self.dnet, self.dfac, self.sigma2)

    # -- raw device entry points on (ncols, n) blocks ---------------------
    def _map(self, col_traj, ncols):
        if col_traj is None:
            if self.M != 1 and ncols != self.M:
                raise ValueError("col_traj needed when ncols != number of trajectories")
            if self.M == 1:
                return None
            col_traj = torch.arange(ncols, dtype=torch.int32, device=self.states.device)
        return torch.as_tensor(col_traj, dtype=torch.int32, device=self.states.device)

    def work(self, ncols):
        return torch.empty(int(_lib.lib().edak_work_doubles(_lib.C.byref(self._P), ncols)),
                           dtype=torch.float64, device=self.states.device)

    def sweep_work(self, ncols):
        k = int(_lib.lib().edak_sweep_work_doubles(_lib.C.byref(self._P), ncols))
        return torch.empty(k, dtype=torch.float64, device=self.states.device)

    def dot_tiles(self):
        """Tile count of the p.Hp partials the fused U_B pass can emit."""
        return int(_lib.lib().edak_hessian_dot_tiles(self.n))

    def hessian_cols(self, Z, col_traj=None, ident=0.0, obs_out=None, out=None, work=None,
                     dot_part=None):
        """out = ident * Z + A Z for a (ncols, n) device block; with ident != 0
        and ``dot_part`` (ncols, dot_tiles()) also the tile partials of
        Z[c].out[c] (PCG p.Hp) from the last U_B pass's epilogue."""
        Z = Z.contiguous()
        ncols = Z.shape[0]
        ct = self._map(col_traj, ncols)
        out = torch.empty_like(Z) if out is None else out
        work = self.work(ncols) if work is None else work
        _lib.call("edak_hessian_block", _lib.C.byref(self._P), Z.data_ptr(), out.data_ptr(),
                  ncols, _lib.ptr(ct), float(ident), work.data_ptr(), _lib.ptr(obs_out),
                  _lib.ptr(dot_part), _lib.stream())
        return out

    def rhs_cols(self, D, col_traj=None, out=None):
        """U_B^T G^T R^-1 d for a (ncols, p) block of innovations (into
        ``out`` (ncols, n), a contiguous block, when given)."""
        D = D.contiguous()
        ncols = D.shape[0]
        ct = self._map(col_traj, ncols)
        if out is None:
            out = torch.empty((ncols, self.n), dtype=torch.float64, device=D.device)
        work = torch.empty((3 * ncols, self.n), dtype=torch.float64, device=D.device)
        _lib.call("edak_rhs", _lib.C.byref(self._P), D.data_ptr(), out.data_ptr(), ncols,
                  _lib.ptr(ct), work.data_ptr(), _lib.stream())
        return out

    def cost_cols(self, Z, D, col_traj=None):
        """J(z) per column against innovations D (ncols, p)."""
        Z, D = Z.contiguous(), D.contiguous()
        ncols = Z.shape[0]
        ct = self._map(col_traj, ncols)
        J = torch.empty(ncols, dtype=torch.float64, device=Z.device)
        _lib.call("edak_cost", _lib.C.byref(self._P), Z.data_ptr(), D.data_ptr(), J.data_ptr(),
                  ncols, _lib.ptr(ct), self.work(ncols).data_ptr(), _lib.stream())
        return J

    def tl_cols(self, V0, col_traj=None):
        """Raw G v0 (no R^-1) for a (ncols, n) block: (ncols, p)."""
        V0 = V0.contiguous()
        ncols = V0.shape[0]
        ct = self._map(col_traj, ncols)
        obs = torch.empty((ncols, self.p), dtype=torch.float64, device=V0.device)
        _lib.call("edak_tl_sweep", _lib.C.byref(self._P), V0.data_ptr(), obs.data_ptr(), ncols,
                  _lib.ptr(ct), self.sweep_work(ncols).data_ptr(), _lib.stream())
        return obs

    def ad_cols(self, W, col_traj=None):
        """G^T (w / sigma^2) for a (ncols, p) block: (ncols, n)."""
        W = W.contiguous()
        ncols = W.shape[0]
        ct = self._map(col_traj, ncols)
        g = torch.empty((ncols, self.n), dtype=torch.float64, device=W.device)
        _lib.call("edak_ad_sweep", _lib.C.byref(self._P), W.data_ptr(), g.data_ptr(), ncols,
                  _lib.ptr(ct), self.sweep_work(ncols).data_ptr(), _lib.stream())
        return g


class MemberProblem:
    """Drop-in for the reference MemberProblem (assim.py:22-85) on the GPU.

    Parameters are the reference's: traj (``.states``, ``.stages``, ``.dt``,
    ``.forcing``), net (``.grid``, ``.times``), ub (``.n``, ``.symbol``),
    rn (``.sigma``), innovation (p,).  ``stage_mode`` ("auto" by default)
    verifies once that the stored stages are recomputable from the states
    and then keeps only the states on the device."""

    def __init__(self, traj, net, ub, rn, innovation, stage_mode="auto"):
        self.traj = traj
        self.net = net
        self.ub = ub
        self.rn = rn
        self.innovation = np.asarray(innovation, dtype=float)
        self.n_matvecs = 0
        stages = getattr(traj, "stages", None)
        self.lin = Linearization(np.asarray(traj.states)[None], traj.dt, traj.forcing, net,
                                 ub, rn, None if stages is None else np.asarray(stages)[None],
                                 stage_mode)
        self._index = None
        self._d = _dev.f64(self.innovation)[None]

    @classmethod
    def view(cls, lin, index, innovation, traj=None):
        """A member on trajectory ``index`` of a shared device Linearization
        (no host trajectory upload; eda.build_setup).  ``innovation`` may be
        a device row; ``traj`` is the reference-style Trajectory (lazy)."""
        self = cls.__new__(cls)
        self.lin = lin
        self.net, self.ub, self.rn = lin.net, lin.ub, lin.rn
        self.traj = traj
        self._index = int(index)
        self._d = torch.as_tensor(innovation, dtype=torch.float64).to(lin.states.device)
        self._d = self._d.reshape(1, -1).contiguous()
        self._innov = None
        self.n_matvecs = 0
        return self

    def __getattr__(self, name):  # lazy host copy for device views
        if name == "innovation":
            self.innovation = self._d[0].cpu().numpy()
            return self.innovation
        raise AttributeError(name)

    def _ct(self, ncols):
        if self._index is None:
            return None
        return torch.full((ncols,), self._index, dtype=torch.int32, device=self.lin.states.device)

    @property
    def n(self):
        return self.lin.n

    @property
    def p(self):
        return self.lin.p

    def a_apply_cols(self, Z):
        """A on a (ncols, n) device block (no host copies); counts one matvec."""
        self.n_matvecs += 1
        return self.lin.hessian_cols(Z, self._ct(Z.shape[0]))

    def a_apply(self, z):
        """A z for (n,) or (n, l); one call = one matvec (assim.py:55-64)."""
        self.n_matvecs += 1
        cols, vec, as_np = _dev.to_cols(z, self.n)
        return _dev.from_cols(self.lin.hessian_cols(cols, self._ct(cols.shape[0])), vec, as_np)

    def hessian_apply(self, z):
        """(I + A) z (assim.py:70-72), the identity fused into the last U_B."""
        self.n_matvecs += 1
        cols, vec, as_np = _dev.to_cols(z, self.n)
        return _dev.from_cols(self.lin.hessian_cols(cols, self._ct(cols.shape[0]), ident=1.0),
                              vec, as_np)

    def hessian_cols(self, Z, ident=1.0, out=None, work=None, dot_part=None):
        """(ident I + A) on a (ncols, n) device block (PCG drop-in path)."""
        return self.lin.hessian_cols(Z, self._ct(Z.shape[0]), ident, None, out, work, dot_part)

    def rhs(self):
        """b = U_B^T G^T R^-1 d (assim.py:74-77)."""
        return self.lin.rhs_cols(self._d, self._ct(1))[0].cpu().numpy()

    def quadratic_cost(self, z):
        """J(z), a TL sweep, not counted as a matvec (assim.py:79-82)."""
        cols, _, _ = _dev.to_cols(z, self.n)
        D = self._d.expand(cols.shape[0], -1)
        return float(self.lin.cost_cols(cols, D, self._ct(cols.shape[0]))[0])

    def reset_matvecs(self):
        self.n_matvecs = 0


def dense_hessian_term(prob):
    """Materialised A (assim.py:88-91)."""
    return prob.a_apply(np.eye(prob.n))


class TrajectoryOperator:
    """A restricted to one trajectory of a multi-trajectory Linearization
    (e.g. the control inside an ensemble): the a_apply duck type that
    nystrom_evd / pcg consume, every column on trajectory ``index``."""

    def __init__(self, lin, index=0):
        self.lin = lin
        self.index = int(index)
        self.n_matvecs = 0

    @property
    def n(self):
        return self.lin.n

    def _ct(self, ncols):
        return torch.full((ncols,), self.index, dtype=torch.int32, device=self.lin.states.device)

    def a_apply_cols(self, Z):
        self.n_matvecs += 1
        return self.lin.hessian_cols(Z, self._ct(Z.shape[0]))

    def a_apply(self, z):
        cols, vec, as_np = _dev.to_cols(z, self.n)
        return _dev.from_cols(self.a_apply_cols(cols), vec, as_np)

    def hessian_apply(self, z):
        self.n_matvecs += 1
        cols, vec, as_np = _dev.to_cols(z, self.n)
        return _dev.from_cols(self.lin.hessian_cols(cols, self._ct(cols.shape[0]), 1.0),
                              vec, as_np)

    def hessian_cols(self, Z, ident=1.0, out=None, work=None, dot_part=None):
        return self.lin.hessian_cols(Z, self._ct(Z.shape[0]), ident, None, out, work, dot_part)


class Ensemble:
    """A batch of members sharing (n, N, dt, F, net, U_B, R).

    Member j owns innovation d_j and linearization trajectory traj_of[j]
    (shared-control mode: every member maps to the control trajectory,
    eda.py:106).  All per-member work is one launch over all columns."""

    def __init__(self, lin, innovations, traj_of=None, control=None):
        self.lin = lin
        self.D = torch.as_tensor(innovations, dtype=torch.float64).to(_dev.device()).contiguous()
        self.M = self.D.shape[0]
        if traj_of is None:
            traj_of = np.arange(self.M)
        if isinstance(traj_of, torch.Tensor) and traj_of.device == self.D.device:
            self.traj_of = traj_of.to(torch.int32).contiguous()  # no host round trip
        else:
            self.traj_of = torch.as_tensor(np.asarray(traj_of), dtype=torch.int32,
                                           device=self.D.device)
        self.control = control  # optional (traj index, innovation row) of the control
        self.n_matvecs = 0

    @property
    def n(self):
        return self.lin.n

    @classmethod
    def from_members(cls, members, stage_mode="auto"):
        """Stack reference-style MemberProblems (identical net/ub/rn/dt).
        Views of one device Linearization (eda.build_setup) are batched
        without touching the host."""
        m0 = members[0]
        lin0 = getattr(m0, "lin", None)
        if lin0 is not None and all(getattr(m, "lin", None) is lin0 and
                                    getattr(m, "_index", None) is not None for m in members):
            D = torch.cat([m._d for m in members], 0)
            return cls(lin0, D, [m._index for m in members])
        trajs, index, traj_of = [], {}, []
        for m in members:
            key = id(m.traj)
            if key not in index:
                index[key] = len(trajs)
                trajs.append(m.traj)
            traj_of.append(index[key])
        states = np.stack([np.asarray(t.states) for t in trajs])
        stages = (np.stack([np.asarray(t.stages) for t in trajs])
                  if getattr(m0.traj, "stages", None) is not None else None)
        lin = Linearization(states, m0.traj.dt, m0.traj.forcing, m0.net, m0.ub, m0.rn,
                            stages, stage_mode)
        innov = np.stack([np.asarray(m.innovation, dtype=float) for m in members])
        return cls(lin, innov, traj_of)

    def subset(self, lo, hi):
        """Members lo..hi-1 as an Ensemble on the same Linearization (device
        views only: safe inside CUDA-graph capture)."""
        return Ensemble(self.lin, self.D[lo:hi], self.traj_of[lo:hi])

    def rhs_all(self, out=None):
        """All members' right-hand sides, (M, n) device block (one launch)."""
        return self.lin.rhs_cols(self.D, self.traj_of, out)

    def a_apply_members(self, Z, ident=0.0, obs_out=None, out=None, work=None, dot_part=None):
        """Column j of Z through member j's Hessian term: (M, n) -> (M, n)."""
        self.n_matvecs += 1
        return self.lin.hessian_cols(Z, self.traj_of, ident, obs_out, out, work, dot_part)

    def cost_members(self, Z):
        return self.lin.cost_cols(Z, self.D, self.traj_of)
