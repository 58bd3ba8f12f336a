"""Twin-experiment construction (restates reference ``eda.py``) and the
BASELINE.json config builders.

``build_setup`` reproduces ``eda.build_setup`` (eda.py:68-109) stream for
stream, so the reference's harness fixtures can be regenerated from this
restatement.  ``baseline_config(i)`` builds config i of BASELINE.json with
the adapters SURVEY.md §8.0 lists: Gaussian B, deterministic truth, and
the obs-time convention ``range(k_t, N+1, k_t)`` (t = 0 excluded).
"""

from dataclasses import dataclass, field

import numpy as np

from . import l96
from .cov import DiagonalNoise, diffusion_factor, gaussian_factor
from .obs import ObsNetwork, strided_grid
from .problem import MemberProblem
from .streams import substream


@dataclass
class TwinConfig:
    """eda.py:31-51 (defaults are the paper headline values)."""

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
    """eda.py:54-65."""

    cfg: object
    net: ObsNetwork
    ub: object
    rn: DiagonalNoise
    truth: l96.Trajectory
    y: np.ndarray
    control: MemberProblem
    members: list = field(default_factory=list)


def _members(cfg, net, ub, rn, y, x_bg, control_traj, trial_seed, shared):
    # eda.py:99-108: member j perturbs background and observations with its
    # own ("bg", j) / ("obsnoise", j) streams; innovation against its own run.
    out = []
    for j in range(1, cfg.members + 1):
        x_j = x_bg + ub.apply(substream(trial_seed, "bg", j).standard_normal(cfg.n))
        y_j = y + rn.apply(substream(trial_seed, "obsnoise", j).standard_normal(net.p))
        traj_j = l96.integrate(x_j, cfg.dt, cfg.n_steps, cfg.forcing)
        lin = control_traj if shared else traj_j
        out.append(MemberProblem(lin, net, ub, rn, y_j - net.observe(traj_j)))
    return out


def build_setup(cfg, trial_seed=None, shared_linearization=False):
    """eda.py:68-109 with the reference's diffusion factor."""
    if trial_seed is None:
        trial_seed = cfg.seed
    net = ObsNetwork(strided_grid(cfg.n, cfg.obs_grid_count), cfg.obs_times)
    ub = diffusion_factor(cfg.n, cfg.sigma_bg, cfg.cov_length, cfg.cov_passes)
    rn = DiagonalNoise(cfg.sigma_obs)
    x_true = l96.spinup(cfg.n, cfg.dt, cfg.forcing, cfg.spinup_steps,
                        substream(cfg.seed, "spinup"))
    truth = l96.integrate(x_true, cfg.dt, cfg.n_steps, cfg.forcing)
    y = net.observe(truth) + rn.apply(substream(cfg.seed, "obsnoise").standard_normal(net.p))
    x_bg = x_true + ub.apply(substream(cfg.seed, "bg", 0).standard_normal(cfg.n))
    control_traj = l96.integrate(x_bg, cfg.dt, cfg.n_steps, cfg.forcing)
    control = MemberProblem(control_traj, net, ub, rn, y - net.observe(control_traj))
    members = _members(cfg, net, ub, rn, y, x_bg, control_traj, trial_seed,
                       shared_linearization)
    return EnsembleSetup(cfg, net, ub, rn, truth, y, control, members)


# --------------------------------------------------- BASELINE.json configs


@dataclass
class BaselineConfig:
    """One row of SURVEY.md §8.0."""

    name: str
    n: int
    n_steps: int
    obs_stride: int          # every k-th variable observed
    obs_every: int           # every k_t-th step observed, t = 0 excluded
    cov_length: float        # Gaussian L in grid points
    members: int
    shared_linearization: bool
    ell: int                 # sketch width
    k: int                   # LMP rank
    pcg_iters: int
    sketch: str = "rhsdiff"  # "rhsdiff" | "rhsdiff+gaussian" | "gaussian"
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

    @property
    def p(self):
        return self.grid_count * len(self.obs_times)


BASELINE_CONFIGS = {
    1: BaselineConfig("cfg1", 40, 8, 2, 1, 2.0, 10, True, 10, 10, 30),
    2: BaselineConfig("cfg2", 40, 8, 2, 1, 2.0, 50, False, 50, 50, 50),
    3: BaselineConfig("cfg3", 1024, 16, 4, 2, 8.0, 50, False, 64, 64, 60,
                      sketch="rhsdiff+gaussian"),
    4: BaselineConfig("cfg4", 16384, 24, 4, 3, 16.0, 200, False, 128, 128, 80),
    5: BaselineConfig("cfg5", 262144, 12, 8, 1, 32.0, 256, False, 256, 128, 20,
                      sketch="rhsdiff"),
}


@dataclass
class BaselineInputs:
    """Host-side inputs of one BASELINE config (the oracle's view)."""

    cfg: BaselineConfig
    net: ObsNetwork
    ub: object
    rn: DiagonalNoise
    x_true: np.ndarray
    y: np.ndarray
    x_bg: np.ndarray
    member_x0: np.ndarray     # (members, n) initial states of member runs
    member_y: np.ndarray      # (members, p) perturbed observations


def baseline_inputs(cfg, members=None, truth=None):
    """Seeded initial conditions/observations for a BASELINE config.

    Streams follow eda.py:87-108.  The trajectories themselves are produced
    by ``l96.integrate`` (oracle) or the GPU producer (product), so large
    configs do not have to integrate on the host.  ``truth`` may pass a
    precomputed spun-up truth state (the 2000-step spin-up is the only
    serial O(n * 2000) host cost)."""
    if members is None:
        members = cfg.members
    net = ObsNetwork(strided_grid(cfg.n, cfg.grid_count), cfg.obs_times)
    ub = gaussian_factor(cfg.n, cfg.sigma_bg, cfg.cov_length)
    rn = DiagonalNoise(cfg.sigma_obs)
    x_true = (l96.deterministic_truth(cfg.n, cfg.dt, cfg.forcing, cfg.spinup_steps)
              if truth is None else np.asarray(truth, dtype=float))
    truth_traj = l96.integrate(x_true, cfg.dt, cfg.n_steps, cfg.forcing)
    y = net.observe(truth_traj) + rn.apply(
        substream(cfg.seed, "obsnoise").standard_normal(net.p))
    x_bg = x_true + ub.apply(substream(cfg.seed, "bg", 0).standard_normal(cfg.n))
    mx = np.empty((members, cfg.n))
    my = np.empty((members, net.p))
    for j in range(1, members + 1):
        mx[j - 1] = x_bg + ub.apply(substream(cfg.seed, "bg", j).standard_normal(cfg.n))
        my[j - 1] = y + rn.apply(substream(cfg.seed, "obsnoise", j).standard_normal(net.p))
    return BaselineInputs(cfg, net, ub, rn, x_true, y, x_bg, mx, my)


def baseline_setup(cfg, members=None, truth=None):
    """Full oracle setup (control + members as MemberProblems) for a
    BASELINE config; integrates every member on the host."""
    inp = baseline_inputs(cfg, members, truth)
    ctl = l96.integrate(inp.x_bg, cfg.dt, cfg.n_steps, cfg.forcing)
    control = MemberProblem(ctl, inp.net, inp.ub, inp.rn, inp.y - inp.net.observe(ctl))
    mems = []
    for j in range(inp.member_x0.shape[0]):
        tj = l96.integrate(inp.member_x0[j], cfg.dt, cfg.n_steps, cfg.forcing)
        lin = ctl if cfg.shared_linearization else tj
        mems.append(MemberProblem(lin, inp.net, inp.ub, inp.rn,
                                  inp.member_y[j] - inp.net.observe(tj)))
    truth_traj = l96.integrate(inp.x_true, cfg.dt, cfg.n_steps, cfg.forcing)
    return EnsembleSetup(cfg, inp.net, inp.ub, inp.rn, truth_traj, inp.y, control, mems)


def baseline_sketch(setup, rng=None):
    """Sketch Omega of a BASELINE config (SURVEY.md §8.0 'Omega' column):
    the first ell rhs differences, padded with Gaussian columns from the
    ("sketch",) stream when ell exceeds the ensemble (cfg3)."""
    from .algorithms import SketchMatrix
    cfg = setup.cfg
    b0 = setup.control.rhs()
    cols = [m.rhs() - b0 for m in setup.members[: cfg.ell]]
    extra = cfg.ell - len(cols)
    if extra > 0:
        rng = substream(cfg.seed, "sketch") if rng is None else rng
        g = rng.standard_normal((cfg.n, extra))
        cols.extend(g.T)
    return SketchMatrix(np.column_stack(cols), cfg.sketch, 0)
