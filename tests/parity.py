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


def pcg_envelope(apply_h, b, cfg, precond=None, cost_fn=None, trials=6, seed=7):
    """(reference trace, envelope of |dJ|, envelope of |d resnorm|)."""
    _, ref = oalg.pcg(apply_h, b, cfg, precond=precond, cost_fn=cost_fn)
    rng = np.random.default_rng(seed)
    n = len(ref.cost)
    e_j, e_r = np.zeros(n), np.zeros(n)
    papply = None if precond is None else (precond if callable(precond) else precond.apply)
    for _ in range(trials):
        def h(v):
            return apply_h(v) * (1 + PCG_JITTER * rng.standard_normal(np.shape(v)))

        def pc(v):
            w = v if papply is None else papply(v)
            return w * (1 + PCG_JITTER * rng.standard_normal(np.shape(v)))
        _, tr = oalg.pcg(h, b, cfg, precond=pc, cost_fn=cost_fn)
        m = min(n, len(tr.cost))
        e_j[:m] = np.maximum(e_j[:m], np.abs(np.array(tr.cost[:m]) - ref.cost[:m]))
        e_r[:m] = np.maximum(e_r[:m], np.abs(np.array(tr.resnorm[:m]) - ref.resnorm[:m]))
    return ref, e_j, e_r


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


def lmp_pcg_envelope(op, phi, ncfg, rule, member, cfg, trials=4, seed=321):
    """CPU-vs-CPU spread of a member's LMP-PCG trace (J, resnorm) when the
    LMP itself is built from Y = A Phi perturbed at the 1e-16 level -- two
    legitimate fp64 Nystrom/Cholesky/SVD implementations differ that way
    (LAPACK-stage results are not bit-pinned)."""
    y = op.a_apply(phi)
    lmp = oalg.make_lmp(oalg.nystrom_evd(lambda v: y, phi, ncfg), rule)
    b = member.rhs()
    _, ref = oalg.pcg(member.hessian_apply, b, cfg, precond=lmp, cost_fn=member.quadratic_cost)
    rng = np.random.default_rng(seed)
    n = len(ref.cost)
    e_j, e_r = np.zeros(n), np.zeros(n)
    for _ in range(trials):
        yp = y * (1 + JITTER * rng.standard_normal(y.shape))
        lp = oalg.make_lmp(oalg.nystrom_evd(lambda v: yp, phi, ncfg), rule)
        _, tr = oalg.pcg(member.hessian_apply, b, cfg, precond=lp, cost_fn=member.quadratic_cost)
        m = min(n, len(tr.cost))
        e_j[:m] = np.maximum(e_j[:m], np.abs(np.array(tr.cost[:m]) - ref.cost[:m]))
        e_r[:m] = np.maximum(e_r[:m], np.abs(np.array(tr.resnorm[:m]) - ref.resnorm[:m]))
    return ref, e_j, e_r


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
