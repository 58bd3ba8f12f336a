"""Sketches, randomized Nystrom EVD, spectral LMP and PCG (restates
reference ``sketch.py``, ``nystrom.py``, ``lmp.py``, ``krylov.py``)."""

from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

# --------------------------------------------------------------- sketch.py


@dataclass
class SketchMatrix:
    """Test-matrix columns + build cost in A-applications (sketch.py:30-40)."""

    columns: np.ndarray
    kind: str
    n_build_matvecs: int = 0

    @property
    def ell(self):
        return self.columns.shape[1]


def gaussian_sketch(n, ell, rng):
    """sketch.py:43-45."""
    return SketchMatrix(rng.standard_normal((n, ell)), "gaussian", 0)


def power_sketch(prob, ell, rng):
    """sketch.py:48-51: A times a Gaussian test matrix (one build matvec)."""
    return SketchMatrix(prob.a_apply(rng.standard_normal((prob.n, ell))), "power", 1)


def bcov_sketch(ub, ell, rng):
    """sketch.py:54-57."""
    return SketchMatrix(ub.apply(ub.apply_t(rng.standard_normal((ub.n, ell)))), "bcov", 0)


def bfactor_sketch(ub, ell, rng):
    """sketch.py:60-63."""
    return SketchMatrix(ub.apply_t(rng.standard_normal((ub.n, ell))), "bfactor", 0)


KINDS = ("gaussian", "power", "bcov", "bfactor", "rhsdiff")


def make_sketch(kind, setup, ell, rng):
    """sketch.py:77-97."""
    if kind == "gaussian":
        return gaussian_sketch(setup.cfg.n, ell, rng)
    if kind == "power":
        return power_sketch(setup.control, ell, rng)
    if kind == "bcov":
        return bcov_sketch(setup.ub, ell, rng)
    if kind == "bfactor":
        return bfactor_sketch(setup.ub, ell, rng)
    if kind == "rhsdiff":
        if ell != len(setup.members):
            raise ValueError(f"rhsdiff sketch width is the ensemble size "
                             f"({len(setup.members)}), got ell={ell}")
        return rhs_diff_sketch(setup.control, setup.members)
    raise ValueError(f"unknown sketch kind {kind!r}; expected one of {KINDS}")


def rhs_diff_sketch(control, members):
    """Gamma_j = b_j - b_0, free in matvecs (sketch.py:66-74)."""
    b0 = control.rhs()
    return SketchMatrix(np.column_stack([m.rhs() - b0 for m in members]),
                        "rhsdiff", 0)


# ------------------------------------------------------------- nystrom.py


class NystromBreakdownError(RuntimeError):
    """nystrom.py:31."""


SHIFT_MODES = (None, "trace", "ynorm")


@dataclass
class NystromConfig:
    """nystrom.py:35-50."""

    ell: int
    k: int
    q: int = 1
    shift_mode: str | None = None

    def __post_init__(self):
        if not 1 <= self.k <= self.ell:
            raise ValueError(f"need 1 <= k <= ell, got k={self.k} ell={self.ell}")
        if self.q < 1:
            raise ValueError(f"need q >= 1, got {self.q}")
        if self.shift_mode not in SHIFT_MODES:
            raise ValueError(f"shift_mode must be one of {SHIFT_MODES}")


@dataclass
class EigenApproximation:
    """nystrom.py:53-64."""

    vectors: np.ndarray
    values: np.ndarray
    shift: float = 0.0
    n_build_matvecs: int = 0

    @property
    def k(self):
        return self.values.size


def shifted_cholesky(w, mode, scale):
    """Plain upper Cholesky, then nu = eps*scale grown x10, at most 5 tries
    (nystrom.py:67-93)."""
    try:
        return scipy.linalg.cholesky(w, lower=False), 0.0
    except scipy.linalg.LinAlgError:
        pass
    nu = np.finfo(float).eps * scale
    if mode is None or nu <= 0.0:
        raise NystromBreakdownError(
            "Cholesky of the sketched Gram matrix broke down and no "
            "usable shift is available")
    eye = np.eye(w.shape[0])
    for _ in range(5):
        try:
            return scipy.linalg.cholesky(w + nu * eye, lower=False), nu
        except scipy.linalg.LinAlgError:
            nu *= 10.0
    raise NystromBreakdownError("sketched Gram matrix stayed indefinite after shifting")


def check_rank(r):
    """nystrom.py:136-140."""
    dead = np.flatnonzero(np.diag(r) == 0.0)
    if dead.size:
        raise NystromBreakdownError(
            f"sketch column {dead[0]} was annihilated by the operator")


def nystrom_evd(a_apply, sketch, cfg):
    """Q-pass randomized Nystrom EVD (nystrom.py:96-133)."""
    phi = np.asarray(getattr(sketch, "columns", sketch), dtype=float)
    if phi.shape[1] != cfg.ell:
        raise ValueError(f"sketch has {phi.shape[1]} columns, cfg.ell={cfg.ell}")
    y = a_apply(phi)
    q_y, r_y = np.linalg.qr(y)
    check_rank(r_y)
    for _ in range(cfg.q - 1):
        phi = q_y
        y = a_apply(phi)
        q_y, r_y = np.linalg.qr(y)
        check_rank(r_y)
    w = phi.T @ y
    scale = np.trace(w) if cfg.shift_mode == "trace" else np.linalg.norm(y)
    c, nu = shifted_cholesky(w, cfg.shift_mode, scale)
    t = scipy.linalg.solve_triangular(c, r_y.T, trans="T", lower=False).T
    u_t, sig, _ = np.linalg.svd(t, full_matrices=False)
    return EigenApproximation(q_y @ u_t[:, :cfg.k], sig[:cfg.k] ** 2, nu, cfg.q)


def reconstruct(approx):
    """S diag(D) S^T (nystrom.py:143-145)."""
    return (approx.vectors * approx.values) @ approx.vectors.T


# ----------------------------------------------------------------- lmp.py

THETA_RULES = ("halfsum", "lambdak", "one")


def choose_theta(rule, lam_k_of_system):
    """lmp.py:25-41."""
    if lam_k_of_system < 1.0 - 1e-8:
        raise ValueError(f"I + A has eigenvalues >= 1, got lam_k={lam_k_of_system}")
    if rule == "halfsum":
        return 0.5 * (lam_k_of_system + 1.0)
    if rule == "lambdak":
        return float(lam_k_of_system)
    if rule == "one":
        return 1.0
    raise ValueError(f"unknown theta rule {rule!r}; expected {THETA_RULES}")


@dataclass
class SpectralLmp:
    """P = U U, U = I + S diag(sqrt(theta/(lam+1)) - 1) S^T (lmp.py:44-74)."""

    vectors: np.ndarray
    values: np.ndarray
    theta: float

    def __post_init__(self):
        if self.theta <= 0:
            raise ValueError("theta must be positive")
        if np.any(self.values < -1e-12):
            raise ValueError("eigenvalue estimates of A must be >= 0")

    @property
    def k(self):
        return self.values.size

    def _project(self, coef, v):
        w = self.vectors.T @ v
        w = coef[:, None] * w if w.ndim == 2 else coef * w
        return v + self.vectors @ w

    def apply_sqrt(self, v):
        return self._project(np.sqrt(self.theta / (self.values + 1.0)) - 1.0, v)

    def apply(self, v):
        return self.apply_sqrt(self.apply_sqrt(v))


def make_lmp(approx, rule):
    """lmp.py:77-81."""
    theta = choose_theta(rule, float(approx.values[-1]) + 1.0)
    return SpectralLmp(approx.vectors, approx.values, theta)


# -------------------------------------------------------------- krylov.py


@dataclass
class SolverConfig:
    """krylov.py:25-37."""

    max_iters: int = 40
    residual_rtol: float | None = None
    trace_cost: bool = True

    def __post_init__(self):
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclass
class SolveTrace:
    """krylov.py:40-46."""

    iterations: list = field(default_factory=list)
    cost: list = field(default_factory=list)
    resnorm: list = field(default_factory=list)
    matvecs: list = field(default_factory=list)
    status: str = "max_iters"


def _as_apply(precond):
    """krylov.py:100-105."""
    if precond is None:
        return lambda v: v
    if callable(precond):
        return precond
    return precond.apply


def _record(trace, it, x, rz, matvecs, cfg, cost_fn):
    """krylov.py:108-113."""
    trace.iterations.append(it)
    trace.cost.append(float(cost_fn(x)) if (cfg.trace_cost and cost_fn) else np.nan)
    trace.resnorm.append(float(np.sqrt(max(rz, 0.0))))
    trace.matvecs.append(matvecs)


def pcg(apply_h, b, cfg, precond=None, cost_fn=None, on_iterate=None):
    """PCG from x0 = 0 with a fixed budget (krylov.py:49-97).

    ``on_iterate(it, x, r, p, rz)`` (oracle-only hook, not in the reference)
    exposes the state after each iteration for teacher-forced parity tests.
    """
    apply_p = _as_apply(precond)
    x = np.zeros_like(b)
    r = b.astype(float).copy()
    z = apply_p(r)
    rz = r @ z
    if rz < 0:
        raise RuntimeError("preconditioner is not positive definite")
    trace = SolveTrace()
    _record(trace, 0, x, rz, 0, cfg, cost_fn)
    rz0 = rz
    p = z
    for it in range(1, cfg.max_iters + 1):
        hp = apply_h(p)
        php = p @ hp
        if php <= 0:
            raise RuntimeError(f"system matrix is not positive definite (iteration {it})")
        alpha = rz / php
        x = x + alpha * p
        r = r - alpha * hp
        z = apply_p(r)
        rz_new = r @ z
        _record(trace, it, x, rz_new, it, cfg, cost_fn)
        if rz_new <= 0 or (cfg.residual_rtol is not None
                           and np.sqrt(rz_new) <= cfg.residual_rtol * np.sqrt(rz0)):
            trace.status = "converged"
            break
        p_new = z + (rz_new / rz) * p
        if on_iterate is not None:
            on_iterate(it, x, r, p_new, rz_new)
        p = p_new
        rz = rz_new
    return x, trace


def _fresh_vector(rng, basis, j, n):
    """Random unit vector orthogonal to the first j basis vectors
    (krylov.py:171-180)."""
    for _ in range(5):
        v = rng.standard_normal(n)
        for _ in range(2):
            v -= basis[:j].T @ (basis[:j] @ v)
        norm = np.linalg.norm(v)
        if norm > 1e-8 * np.sqrt(n):
            return v / norm
    return None


def lanczos_eigs(apply_h, n, m, n_eigs, seed=0):
    """Lanczos with full reorthogonalization and invariant-subspace restarts
    (krylov.py:116-168)."""
    from .streams import substream
    m = min(m, n)
    if not 1 <= n_eigs <= m:
        raise ValueError("need 1 <= n_eigs <= m")
    rng = substream(seed, "lanczos")
    basis = np.empty((m, n))
    alphas = np.zeros(m)
    betas = np.zeros(m)
    block_end = {}
    basis[0] = _fresh_vector(rng, basis, 0, n)
    scale = 0.0
    j = 0
    while j < m:
        w = apply_h(basis[j])
        alphas[j] = basis[j] @ w
        w -= alphas[j] * basis[j]
        for _ in range(2):
            w -= basis[: j + 1].T @ (basis[: j + 1] @ w)
        beta = np.linalg.norm(w)
        scale = max(scale, abs(alphas[j]), beta)
        if j + 1 == m:
            block_end[j] = beta
            break
        if beta <= 1e-12 * max(scale, 1.0):
            block_end[j] = beta
            nxt = _fresh_vector(rng, basis, j + 1, n)
            if nxt is None:
                m = j + 1
                break
            basis[j + 1] = nxt
        else:
            betas[j] = beta
            basis[j + 1] = w / beta
        j += 1
    tri = np.diag(alphas[:m]) + np.diag(betas[: m - 1], 1) + np.diag(betas[: m - 1], -1)
    theta, s = np.linalg.eigh(tri)
    order = np.argsort(theta)[::-1][:n_eigs]
    bounds = np.array([sum(abs(b * s[pos, i]) for pos, b in block_end.items()) for i in order])
    return theta[order], bounds
