"""CPU restatement of the reference experiment driver (``harness.py``).

TEST INFRASTRUCTURE ONLY: the GPU harness (paper_2605_23571_b200.harness)
is checked against these rows and against the reference's own fixture CSVs
(tests/golden/harness_fixtures.json).  Row order, keys and the matvec
convention follow harness.py:126-267 exactly; ``validate`` is not restated
(it is a self-check that the GPU test runs directly).
"""

from dataclasses import replace

from .algorithms import (NystromConfig, SolverConfig, lanczos_eigs, make_lmp, make_sketch,
                         nystrom_evd, pcg)
from .streams import substream
from .twin import build_setup


def _lanczos_budget(twin):
    """harness.py:120-123."""
    return min(twin.n, twin.p + 80)


def _trace_rows(rows, key, trace, build):
    """harness.py:185-189."""
    for it, cost in zip(trace.iterations, trace.cost):
        rows.append(key + (it, "J", cost))
    for it, mv in zip(trace.iterations, trace.matvecs):
        rows.append(key + (it, "matvecs", build + mv))


def _solve(prob, precond, max_iters):
    """harness.py:178-182."""
    prob.n_matvecs = 0
    return pcg(prob.hessian_apply, prob.rhs(), SolverConfig(max_iters=max_iters),
               precond=precond, cost_fn=prob.quadratic_cost)


def eig_sensitivity(twin, seed, length_grid, passes_grid):
    """harness.py:126-145. Rows (seed, member, variant, rule, k, index, metric, value)."""
    rows = []
    cells = ([("D", L, twin.cov_passes) for L in length_grid]
             + [("M", twin.cov_length, m) for m in passes_grid])
    for axis, length, passes in cells:
        tw = replace(twin, cov_length=length, cov_passes=passes)
        setup = build_setup(tw)
        n_top = min(150, twin.p) if axis == "D" else min(40, twin.p)
        vals, _ = lanczos_eigs(setup.control.hessian_apply, tw.n, _lanczos_budget(tw), n_top,
                               seed=tw.seed)
        label = f"D={length:g}" if axis == "D" else f"M={passes:g}"
        for i, lam in enumerate(vals, start=1):
            rows.append((seed, "", label, "", "", i, "eigenvalue", lam))
    return rows


def eig_error(twin, seeds, kinds, k, ell):
    """harness.py:148-175."""
    rows = []
    oracle_setup = build_setup(twin)
    ref, _ = lanczos_eigs(oracle_setup.control.hessian_apply, twin.n, _lanczos_budget(twin), k,
                          seed=twin.seed)
    for i, lam in enumerate(ref, start=1):
        rows.append((twin.seed, "", "oracle", "", k, i, "eigenvalue", lam))
    ncfg = NystromConfig(ell=ell, k=k, shift_mode="trace")
    for seed in seeds:
        setup = build_setup(twin, trial_seed=seed)
        for kind in kinds:
            sk = make_sketch(kind, setup, ell, substream(seed, "sketch"))
            approx = nystrom_evd(setup.control.a_apply, sk, ncfg)
            for i in range(k):
                err = abs((approx.values[i] + 1.0) - ref[i]) / ref[i]
                rows.append((seed, "", kind, "", k, i + 1, "rel_error", err))
    return rows


def control_lmp(twin, seeds, kinds, rule, k, ell, max_iters):
    """harness.py:192-214."""
    rows = []
    ncfg = NystromConfig(ell=ell, k=k, shift_mode="trace")
    for seed in seeds:
        setup = build_setup(twin, trial_seed=seed)
        _, tr = _solve(setup.control, None, max_iters)
        _trace_rows(rows, (seed, "", "none", "", ""), tr, 0)
        for kind in kinds:
            sk = make_sketch(kind, setup, ell, substream(seed, "sketch"))
            approx = nystrom_evd(setup.control.a_apply, sk, ncfg)
            _, tr = _solve(setup.control, make_lmp(approx, rule), max_iters)
            _trace_rows(rows, (seed, "", kind, rule, k), tr, sk.n_build_matvecs + 1)
    return rows


def theta_sensitivity(twin, seeds, kind, rules, k_list, ell, max_iters):
    """harness.py:217-238."""
    rows = []
    for seed in seeds:
        setup = build_setup(twin, trial_seed=seed)
        _, tr = _solve(setup.control, None, max_iters)
        _trace_rows(rows, (seed, "", "none", "", ""), tr, 0)
        sk = make_sketch(kind, setup, ell, substream(seed, "sketch"))
        for k in k_list:
            approx = nystrom_evd(setup.control.a_apply, sk,
                                 NystromConfig(ell=ell, k=k, shift_mode="trace"))
            for rule in rules:
                _, tr = _solve(setup.control, make_lmp(approx, rule), max_iters)
                _trace_rows(rows, (seed, "", kind, rule, k), tr, sk.n_build_matvecs + 1)
    return rows


def ensemble_lmp(twin, seed, kind, rule, k_list, ell, max_iters):
    """harness.py:241-267."""
    rows = []
    setup = build_setup(twin, trial_seed=seed)
    sk = make_sketch(kind, setup, ell, substream(seed, "sketch"))
    plain = []
    for j, m in enumerate(setup.members, start=1):
        _, tr = _solve(m, None, max_iters)
        plain.append(tr)
        _trace_rows(rows, (seed, j, "none", "", ""), tr, 0)
    for k in k_list:
        approx = nystrom_evd(setup.control.a_apply, sk,
                             NystromConfig(ell=ell, k=k, shift_mode="trace"))
        lmp = make_lmp(approx, rule)
        for j, m in enumerate(setup.members, start=1):
            _, tr = _solve(m, lmp, max_iters)
            key = (seed, j, kind, rule, k)
            _trace_rows(rows, key, tr, sk.n_build_matvecs + 1)
            for it, (a, b) in enumerate(zip(plain[j - 1].cost, tr.cost)):
                rows.append(key + (it, "J_ratio", a / b))
    return rows
