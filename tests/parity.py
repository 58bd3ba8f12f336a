"""Parity protocol helpers.

Some reference outputs are ill-conditioned functions of the operator: two
legitimate fp64 evaluations of A differ by ~1e-16 per apply, and late PCG
iterates or the smallest Nystrom values of an ill-conditioned sketch move by
far more than 1e-10 under such perturbations *on the CPU itself*.  These
helpers measure that CPU-vs-CPU envelope with the oracle in the same test
(apply_h / Y multiplied by (1 + 2e-16 xi), xi ~ N(0,1)), and the GPU result
must lie within max(rel 1e-10 of the reference, 10 x envelope).
"""

import numpy as np

from oracle import algorithms as oalg

JITTER = 2e-16
# PCG envelope: two legitimate fp64 PCG implementations differ in the operator
# (~1e-16 per element) AND in every dot product's summation order (relative
# error ~ sqrt(n) eps); both are emulated by jittering H p and P r at 1e-15.
PCG_JITTER = 1e-15


class _ScipyFftFactor:
    """The oracle's circulant factor with scipy.fft (pypocketfft) in place
    of numpy.fft: an equally valid fp64 evaluation of covariance.py:41-45
    that rounds differently ('oracle with numpy.fft vs
    scipy.fft')."""

    def __init__(self, ub):
        self.n, self.symbol = ub.n, ub.symbol

    def apply(self, v):
        import scipy.fft as sfft
        vhat = sfft.rfft(v, axis=0)
        vhat *= self.symbol[:, None] if vhat.ndim == 2 else self.symbol
        return sfft.irfft(vhat, n=self.n, axis=0)

    apply_t = apply


def _single_pass(lmp):
    """P v = v + S diag(theta/(lam+1) - 1) S^T v: the one-pass form of the
    reference's P = U(U v) (lmp.py:72-74), equal in exact arithmetic."""
    S, c = lmp.vectors, lmp.theta / (lmp.values + 1.0) - 1.0

    def apply(v):
        w = S.T @ v
        return v + S @ ((c[:, None] * w) if w.ndim == 2 else c * w)
    return apply


def _variants(apply_h, precond, cost_fn):
    """Structured CPU-vs-CPU variants of one PCG solve, each a legitimate
    fp64 implementation of the reference algorithm: the one-pass LMP, the
    scipy.fft factor, and both.  Measured at cfg4: a PCG stagnation bump
    (iterations ~20-25) amplifies the one-pass/two-pass difference to
    2.7e-7 relative in J, ~10x more than random 1e-15 jitter shows."""
    out = []
    prob = getattr(apply_h, "__self__", None)
    alt = None
    if prob is not None and getattr(apply_h, "__name__", "") == "hessian_apply" and hasattr(prob, "ub"):
        from oracle.problem import MemberProblem
        alt = MemberProblem(prob.traj, prob.net, _ScipyFftFactor(prob.ub), prob.rn, prob.innovation)
    alt_cost = None
    if alt is not None and cost_fn is not None and getattr(cost_fn, "__self__", None) is prob:
        alt_cost = alt.quadratic_cost
    one = _single_pass(precond) if isinstance(precond, oalg.SpectralLmp) else None
    if one is not None:
        out.append((apply_h, one, cost_fn))
    if alt is not None and (cost_fn is None or alt_cost is not None):
        out.append((alt.hessian_apply, precond, alt_cost))
        if one is not None:
            out.append((alt.hessian_apply, one, alt_cost))
    return out


def pcg_envelope(apply_h, b, cfg, precond=None, cost_fn=None, trials=6, seed=7, with_x=False):
    """(reference trace, envelope of |dJ|, envelope of |d resnorm|); with
    ``with_x`` also (reference x, envelope of ||dx||).  The envelope is the
    spread over random 1e-15 jitter of H p and P r (``trials`` runs) and the
    structured variants of ``_variants``."""
    x_ref, ref = oalg.pcg(apply_h, b, cfg, precond=precond, cost_fn=cost_fn)
    rng = np.random.default_rng(seed)
    n = len(ref.cost)
    e_j, e_r, e_x = np.zeros(n), np.zeros(n), 0.0
    papply = None if precond is None else (precond if callable(precond) else precond.apply)
    one = _single_pass(precond) if isinstance(precond, oalg.SpectralLmp) else None
    runs = []
    for t in range(trials):
        # jitter on top of the two-pass and (alternately) the one-pass LMP
        base = one if (one is not None and t % 2) else papply

        def h(v):
            return apply_h(v) * (1 + PCG_JITTER * rng.standard_normal(np.shape(v)))

        def pc(v, base=base):
            w = v if base is None else base(v)
            return w * (1 + PCG_JITTER * rng.standard_normal(np.shape(v)))
        runs.append((h, pc, cost_fn))
    runs.extend(_variants(apply_h, precond, cost_fn))
    for h, pc, cf in runs:
        x, tr = oalg.pcg(h, b, cfg, precond=pc, cost_fn=cf)
        m = min(n, len(tr.cost))
        e_j[:m] = np.maximum(e_j[:m], np.abs(np.array(tr.cost[:m]) - ref.cost[:m]))
        e_r[:m] = np.maximum(e_r[:m], np.abs(np.array(tr.resnorm[:m]) - ref.resnorm[:m]))
        e_x = max(e_x, float(np.linalg.norm(x - x_ref)))
    if with_x:
        return ref, e_j, e_r, x_ref, e_x
    return ref, e_j, e_r


def assert_increment(x, x_ref, env_x, rtol=1e-10):
    """Final increment (krylov.py:97): ||x - x_ref|| <= max(rtol ||x_ref||,
    10 x the CPU-vs-CPU spread of x)."""
    x, x_ref = np.asarray(x), np.asarray(x_ref)
    err = float(np.linalg.norm(x - x_ref))
    tol = max(rtol * float(np.linalg.norm(x_ref)), 10.0 * env_x)
    assert err <= tol, ("x", err, tol, float(np.linalg.norm(x_ref)))
    return err / float(np.linalg.norm(x_ref))


def assert_trace(ours, ref, env_j, env_r, rtol=1e-10):
    """J within rel 1e-10 or 10x envelope at every iteration; resnorm within
    1e-10 r0 up to the divergence onset (the first iteration where 10x the
    CPU-vs-CPU resnorm envelope exceeds 1e-10 r0 -- the same 10x margin as J,
    since a 3-trial envelope underestimates the spread of a different but
    equally valid rounding order).  Past the onset the residual history
    is round-off chaotic (SURVEY.md §7 hard part 1) and step-level exactness
    is checked by the teacher-forced test instead."""
    assert len(ours.cost) == len(ref.cost), (len(ours.cost), len(ref.cost))
    J, Jr = np.asarray(ours.cost), np.asarray(ref.cost)
    tol = np.maximum(rtol * np.abs(Jr), 10 * env_j)
    bad = np.abs(J - Jr) > tol
    assert not bad.any(), ("J", np.flatnonzero(bad), J[bad], Jr[bad], tol[bad])
    R, Rr = np.asarray(ours.resnorm), np.asarray(ref.resnorm)
    onset = np.flatnonzero(10 * env_r > rtol * Rr[0])
    upto = onset[0] if onset.size else len(Rr)
    tol = np.full(len(Rr), rtol * Rr[0])
    bad = (np.abs(R - Rr) > tol) & (np.arange(len(Rr)) < upto)
    assert not bad.any(), ("resnorm", np.flatnonzero(bad), R[bad], Rr[bad], tol[bad])


def nystrom_envelope(op, phi, cfg, trials=4):
    """Per-value CPU-vs-CPU spread of the reference Nystrom values when
    Y = A Phi is perturbed at the 1e-16 level."""
    y = op.a_apply(phi)
    base = oalg.nystrom_evd(lambda v: y, phi, cfg).values
    rng = np.random.default_rng(123)
    env = np.zeros_like(base)
    for _ in range(trials):
        yp = y * (1 + JITTER * rng.standard_normal(y.shape))
        env = np.maximum(env, np.abs(oalg.nystrom_evd(lambda v: yp, phi, cfg).values - base))
    return env


def lmp_pcg_envelope(op, phi, ncfg, rule, member, cfg, trials=4, seed=321, with_x=False):
    """CPU-vs-CPU spread of a member's LMP-PCG trace (J, resnorm; with
    ``with_x`` also the final increment) when the LMP itself is built from
    Y = A Phi perturbed at the 1e-16 level -- two legitimate fp64
    Nystrom/Cholesky/SVD implementations differ that way (SURVEY.md §8c:
    LAPACK-stage results are not bit-pinned)."""
    y = op.a_apply(phi)
    lmp = oalg.make_lmp(oalg.nystrom_evd(lambda v: y, phi, ncfg), rule)
    b = member.rhs()
    x_ref, ref = oalg.pcg(member.hessian_apply, b, cfg, precond=lmp, cost_fn=member.quadratic_cost)
    rng = np.random.default_rng(seed)
    n = len(ref.cost)
    e_j, e_r, e_x = np.zeros(n), np.zeros(n), 0.0
    for _ in range(trials):
        yp = y * (1 + JITTER * rng.standard_normal(y.shape))
        lp = oalg.make_lmp(oalg.nystrom_evd(lambda v: yp, phi, ncfg), rule)
        for pc in (lp, _single_pass(lp)):
            x, tr = oalg.pcg(member.hessian_apply, b, cfg, precond=pc,
                             cost_fn=member.quadratic_cost)
            m = min(n, len(tr.cost))
            e_j[:m] = np.maximum(e_j[:m], np.abs(np.array(tr.cost[:m]) - ref.cost[:m]))
            e_r[:m] = np.maximum(e_r[:m], np.abs(np.array(tr.resnorm[:m]) - ref.resnorm[:m]))
            e_x = max(e_x, float(np.linalg.norm(x - x_ref)))
    if with_x:
        return ref, e_j, e_r, x_ref, e_x
    return ref, e_j, e_r


def nystrom_envelope_y(y, phi, cfg, trials=4):
    """nystrom_envelope for a given Y = A Phi (e.g. the GPU's own Y, so that
    only the dense Nystrom stage is compared): (reference approximation,
    per-value CPU-vs-CPU spread)."""
    base = oalg.nystrom_evd(lambda v: y, phi, cfg)
    rng = np.random.default_rng(123)
    env = np.zeros_like(base.values)
    for _ in range(trials):
        yp = y * (1 + JITTER * rng.standard_normal(y.shape))
        env = np.maximum(env, np.abs(oalg.nystrom_evd(lambda v: yp, phi, cfg).values - base.values))
    return base, env


def assert_values(ours, ref, env):
    """rel 1e-10 for D_i >= 1e-6 D_1, else abs 1e-10 D_1, widened to 10x the
    measured envelope where that is larger."""
    ours, ref = np.asarray(ours), np.asarray(ref)
    tol = np.where(ref >= 1e-6 * ref[0], 1e-10 * np.abs(ref), 1e-10 * ref[0])
    tol = np.maximum(tol, 10.0 * env)
    bad = np.abs(ours - ref) > tol
    assert not bad.any(), (ours[bad], ref[bad], tol[bad])


def teacher_forced_step(apply_h, apply_p, x, r, p, rz):
    """One reference PCG iteration (krylov.py:80-95) from a given state."""
    hp = apply_h(p)
    alpha = rz / (p @ hp)
    x1 = x + alpha * p
    r1 = r - alpha * hp
    z1 = apply_p(r1) if apply_p is not None else r1
    rz1 = r1 @ z1
    return x1, r1, z1 + (rz1 / rz) * p, rz1


def oracle_rows(dens, rows):
    """Oracle MemberProblems for ensemble rows (0 = control) on the device
    ensemble's own trajectories and innovations (only the needed
    trajectories are copied to the host: cfg5's full set is 7 GB)."""
    from oracle import l96 as ol96
    from oracle.cov import CirculantFactor as OFactor, DiagonalNoise as ONoise
    from oracle.obs import ObsNetwork as OObs
    from oracle.problem import MemberProblem as OProblem
    cfg = dens.cfg
    net = OObs(dens.net.grid, dens.net.times)
    ub = OFactor(cfg.n, dens.ub.symbol)
    out, cache = [], {}
    for r in rows:
        t = int(dens.traj_of[r])
        if t not in cache:
            st = dens.states[t].cpu().numpy()
            stg = np.stack([np.stack(ol96.rk4_stages(st[s], cfg.dt, cfg.forcing)[1])
                            for s in range(cfg.n_steps)])
            cache[t] = ol96.Trajectory(st, stg, cfg.dt, cfg.forcing)
        out.append(OProblem(cache[t], net, ub, ONoise(cfg.sigma_obs),
                            dens.innovations[r].cpu().numpy()))
    return out
