"""Generate golden vectors by running the REAL reference (edasketch).

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes ``tests/golden/ref_*.npz`` and ``tests/golden/fixtures.json``.  All
inputs are built with reference functions only (``edasketch.*``); the
BASELINE-config cases compose the reference ``MemberProblem`` /
``ObsNetwork`` / ``model`` with a Gaussian-symbol factor (the reference
``GridCovFactor`` with its ``symbol`` replaced -- the duck type its
``apply`` reads, covariance.py:41-45) as SURVEY.md §8c prescribes.
"""

import csv
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from edasketch import model  # noqa: E402
from edasketch.assim import MemberProblem  # noqa: E402
from edasketch.covariance import DiagonalNoise, GridCovFactor  # noqa: E402
from edasketch.eda import TwinConfig, build_setup  # noqa: E402
from edasketch.krylov import SolverConfig, pcg  # noqa: E402
from edasketch.lmp import make_lmp  # noqa: E402
from edasketch.nystrom import NystromConfig, nystrom_evd  # noqa: E402
from edasketch.obs import ObsNetwork, strided_grid  # noqa: E402
from edasketch.sketch import gaussian_sketch, make_sketch  # noqa: E402
from edasketch.streams import substream  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = "/root/reference/pkg/frontend/test/fixtures"


def gaussian_symbol(n, sigma_b, length):
    # same closed form as oracle/cov.py:gaussian_spectrum (the adapter)
    m = np.arange(n // 2 + 1, dtype=float) / n
    c = np.zeros_like(m)
    for k in range(-3, 4):
        c += np.exp(-2.0 * np.pi ** 2 * length ** 2 * (m - k) ** 2)
    return sigma_b * np.sqrt(np.sqrt(2.0 * np.pi) * length * c)


def gaussian_ub(n, sigma_b, length):
    ub = GridCovFactor(n, sigma_b, 1.0, 1)
    ub.symbol = gaussian_symbol(n, sigma_b, length)
    return ub


def baseline_like(n, n_steps, stride, every, length, members, shared, seed=0,
                  spin=2000):
    """BASELINE-config construction with reference functions only."""
    dt, forcing = 0.025, 8.0
    x = np.full(n, forcing)
    x[0] += 0.01
    for _ in range(spin):
        x = model.rk4_step(x, dt, forcing)
    net = ObsNetwork(strided_grid(n, n // stride), list(range(every, n_steps + 1, every)))
    ub = gaussian_ub(n, 0.8, length)
    rn = DiagonalNoise(1.0)
    truth = model.integrate(x, dt, n_steps, forcing)
    y = net.observe(truth) + rn.apply(substream(seed, "obsnoise").standard_normal(net.p))
    x_bg = x + ub.apply(substream(seed, "bg", 0).standard_normal(n))
    ctl = model.integrate(x_bg, dt, n_steps, forcing)
    control = MemberProblem(ctl, net, ub, rn, y - net.observe(ctl))
    mems = []
    for j in range(1, members + 1):
        xj = x_bg + ub.apply(substream(seed, "bg", j).standard_normal(n))
        yj = y + rn.apply(substream(seed, "obsnoise", j).standard_normal(net.p))
        tj = model.integrate(xj, dt, n_steps, forcing)
        mems.append(MemberProblem(ctl if shared else tj, net, ub, rn, yj - net.observe(tj)))
    return x, control, mems


def pack_problem(prefix, prob, out):
    out[prefix + "states"] = prob.traj.states
    out[prefix + "stages"] = prob.traj.stages
    out[prefix + "innov"] = prob.innovation
    out[prefix + "grid"] = prob.net.grid
    out[prefix + "times"] = prob.net.times
    out[prefix + "symbol"] = prob.ub.symbol
    out[prefix + "sigma_obs"] = np.array(prob.rn.sigma)


def trace_arrays(prefix, tr, out, x=None):
    if x is not None:  # the final increment krylov.pcg returns (krylov.py:97)
        out[prefix + "x"] = np.asarray(x)
    out[prefix + "cost"] = np.array(tr.cost)
    out[prefix + "resnorm"] = np.array(tr.resnorm)
    out[prefix + "iters"] = np.array(tr.iterations)
    out[prefix + "status"] = np.array(tr.status)


def make_model_cases():
    out = {}
    # tendency known answers on random states (model.py:20-35)
    rng = substream(7, "golden", "model")
    x = rng.standard_normal(40) * 3 + 2
    v = rng.standard_normal(40)
    out["x"], out["v"] = x, v
    out["tend"] = model.tendency(x, 8.0)
    out["tend_tl"] = model.tendency_tlm(x, v)
    out["tend_ad"] = model.tendency_adj(x, v)
    traj = model.integrate(x, 0.025, 8, 8.0)
    out["int_states"], out["int_stages"] = traj.states, traj.stages
    out["tlm"] = model.tlm(traj, v)
    w = rng.standard_normal((9, 40))
    out["adj_w"], out["adj"] = w, model.adjoint(traj, w)
    # deterministic truth (BASELINE adapter) at n=40, 2000 steps
    xt = np.full(40, 8.0)
    xt[0] += 0.01
    for _ in range(2000):
        xt = model.rk4_step(xt, 0.025, 8.0)
    out["truth40"] = xt
    # obs network incl. t = 0 (test_obs.py:75-88 pattern)
    net = ObsNetwork([0, 3, 7], [0, 2, 4])
    traj = model.integrate(x[:10], 0.025, 4, 8.0)
    out["obs0_states"], out["obs0_stages"] = traj.states, traj.stages
    out["obs0_y"] = net.observe(traj)
    out["obs0_tl"] = net.observe_tlm(traj, v[:10])
    out["obs0_w"] = w[0, : net.p]
    out["obs0_ad"] = net.observe_adj(traj, w[0, : net.p])
    np.savez_compressed(os.path.join(HERE, "ref_model.npz"), **out)


def make_problem_cases():
    out = {}
    # (1) reference tiny.cfg twin (diffusion B), shared by the fixtures
    tw = TwinConfig(n=40, obs_grid_count=8, members=10)
    setup = build_setup(tw, trial_seed=0)
    prob = setup.control
    pack_problem("tiny_", prob, out)
    z = substream(11, "golden", "z").standard_normal((40, 6))
    out["tiny_z"] = z
    out["tiny_az"] = prob.a_apply(z)
    out["tiny_rhs"] = prob.rhs()
    out["tiny_cost"] = np.array([prob.quadratic_cost(z[:, j]) for j in range(6)])
    out["tiny_dense_a"] = prob.a_apply(np.eye(40))
    x, tr = pcg(prob.hessian_apply, prob.rhs(), SolverConfig(max_iters=8),
                cost_fn=prob.quadratic_cost)
    trace_arrays("tiny_pcg_", tr, out, x)
    sk = make_sketch("rhsdiff", setup, 10, substream(0, "sketch"))
    out["tiny_gamma"] = sk.columns
    out["tiny_member_rhs"] = np.column_stack([m.rhs() for m in setup.members])
    approx = nystrom_evd(prob.a_apply, sk, NystromConfig(ell=10, k=8, shift_mode="trace"))
    out["tiny_nys_vals"], out["tiny_nys_vecs"] = approx.values, approx.vectors
    out["tiny_nys_shift"] = np.array(approx.shift)
    lmp = make_lmp(approx, "halfsum")
    out["tiny_theta"] = np.array(lmp.theta)
    x, tr = pcg(prob.hessian_apply, prob.rhs(), SolverConfig(max_iters=8),
                precond=lmp, cost_fn=prob.quadratic_cost)
    trace_arrays("tiny_lmp_", tr, out, x)

    # (2) BASELINE cfg1-like: n=40, N=8, every 2nd var every step, shared
    x, control, mems = baseline_like(40, 8, 2, 1, 2.0, 10, True)
    out["cfg1_truth"] = x
    pack_problem("cfg1_", control, out)
    out["cfg1_member_innov"] = np.stack([m.innovation for m in mems])
    out["cfg1_member_rhs"] = np.column_stack([m.rhs() for m in mems])
    z = substream(12, "golden", "z").standard_normal((40, 10))
    out["cfg1_z"], out["cfg1_az"] = z, control.a_apply(z)
    b0 = control.rhs()
    gam = np.column_stack([m.rhs() - b0 for m in mems])
    out["cfg1_gamma"] = gam
    approx = nystrom_evd(control.a_apply, gam, NystromConfig(ell=10, k=10, shift_mode="trace"))
    out["cfg1_nys_vals"], out["cfg1_nys_vecs"] = approx.values, approx.vectors
    out["cfg1_nys_shift"] = np.array(approx.shift)
    lmp = make_lmp(approx, "halfsum")
    for j in (0, 4, 9):
        x, tr = pcg(mems[j].hessian_apply, mems[j].rhs(), SolverConfig(max_iters=30),
                    precond=lmp, cost_fn=mems[j].quadratic_cost)
        trace_arrays(f"cfg1_m{j}_", tr, out, x)

    # (3) BASELINE cfg2-like: 50 own trajectories, ell=50 > n (shift path)
    x, control, mems = baseline_like(40, 8, 2, 1, 2.0, 50, False)
    pack_problem("cfg2_", control, out)
    b0 = control.rhs()
    gam = np.column_stack([m.rhs() - b0 for m in mems])
    out["cfg2_gamma"] = gam
    for k in (10, 20, 50):
        approx = nystrom_evd(control.a_apply, gam, NystromConfig(ell=50, k=k, shift_mode="trace"))
        out[f"cfg2_k{k}_vals"], out[f"cfg2_k{k}_vecs"] = approx.values, approx.vectors
        out[f"cfg2_k{k}_shift"] = np.array(approx.shift)
    for j in (0, 17):
        m = mems[j]
        pack_problem(f"cfg2_m{j}_", m, out)
        approx = nystrom_evd(control.a_apply, gam, NystromConfig(ell=50, k=20, shift_mode="trace"))
        x, tr = pcg(m.hessian_apply, m.rhs(), SolverConfig(max_iters=50),
                    precond=make_lmp(approx, "halfsum"), cost_fn=m.quadratic_cost)
        trace_arrays(f"cfg2_m{j}_", tr, out, x)

    # (4) n=120 mirror (test_nystrom.py:21-24) with a gaussian sketch
    tw = TwinConfig(n=120, obs_grid_count=10, members=0, seed=21)
    prob = build_setup(tw).control
    pack_problem("mir_", prob, out)
    sk = gaussian_sketch(120, 20, substream(4, "sk"))
    out["mir_phi"] = sk.columns
    out["mir_y"] = prob.a_apply(sk.columns)
    approx = nystrom_evd(prob.a_apply, sk, NystromConfig(ell=20, k=15, shift_mode="trace"))
    out["mir_nys_vals"], out["mir_nys_vecs"] = approx.values, approx.vectors
    np.savez_compressed(os.path.join(HERE, "ref_problem.npz"), **out)


def extract_fixtures():
    """Pull the harness fixtures' LAPACK-free rows (variant=none J traces,
    SURVEY.md §8c) into JSON so the GPU box does not need the reference."""
    keep = {}
    for name in ("control-lmp", "ensemble-lmp", "theta-sensitivity"):
        rows = {}
        with open(os.path.join(FIXTURES, name + ".csv"), newline="") as fh:
            for row in csv.DictReader(fh):
                if row["variant"] != "none" or row["metric"] != "J":
                    continue
                key = f"{row['seed']}/{row['member']}"
                rows.setdefault(key, []).append((int(row["index"]), row["value"]))
        keep[name] = {k: [v for _, v in sorted(vs)] for k, vs in rows.items()}
    # Lanczos eigenvalues of I + A (eig-sensitivity, harness.py:126-146)
    eig = {}
    with open(os.path.join(FIXTURES, "eig-sensitivity.csv"), newline="") as fh:
        for row in csv.DictReader(fh):
            eig.setdefault(row["variant"], []).append((int(row["index"]), row["value"]))
    keep["eig-sensitivity"] = {k: [v for _, v in sorted(vs)] for k, vs in eig.items()}
    # fixture configs (tiny.cfg / ensemble.cfg / theta.cfg are n=40, G=8,
    # 10 members, 8 iterations; seeds from regenerate.sh)
    keep["config"] = {"n": 40, "obs_grid_count": 8, "members": 10, "max_iters": 8}
    with open(os.path.join(HERE, "fixtures.json"), "w") as fh:
        json.dump(keep, fh, indent=1, sort_keys=True)


def extract_harness_rows():
    """Every row of the reference's fixture CSVs (regenerate.sh: tiny.cfg,
    theta.cfg, ensemble.cfg at n=40), as written by the reference harness,
    for the GPU harness CSV-contract test."""
    out = {}
    for name in ("eig-sensitivity", "eig-error", "control-lmp", "theta-sensitivity",
                 "ensemble-lmp"):
        with open(os.path.join(FIXTURES, name + ".csv"), newline="") as fh:
            rd = csv.reader(fh)
            header = next(rd)
            out[name] = [row for row in rd]
    out["header"] = header
    with open(os.path.join(HERE, "harness_fixtures.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))


def regen_harness_rows():
    """The same five fixture runs regenerated HERE by the unmodified
    reference harness (its own run_experiment): pins the oracle restatement
    bit for bit on this numpy/LAPACK, and |regen - fixture| measures the
    machine-to-machine spread of the LAPACK-stage rows (the GPU tolerance)."""
    from dataclasses import replace as dc_replace
    from edasketch import harness
    specs = {
        "eig-sensitivity": dict(k_list=[8], kinds=["gaussian", "power", "rhsdiff"],
                                length_grid=[2.0, 6.0], passes_grid=[4, 10], seeds=[0]),
        "eig-error": dict(k_list=[8], kinds=["gaussian", "power", "rhsdiff"],
                          length_grid=[2.0, 6.0], passes_grid=[4, 10], seeds=[0, 1, 2]),
        "control-lmp": dict(k_list=[8], kinds=["gaussian", "power", "rhsdiff"],
                            length_grid=[2.0, 6.0], passes_grid=[4, 10], seeds=[0, 1, 2]),
        "theta-sensitivity": dict(k_list=[8, 6], seeds=[0, 1]),
        "ensemble-lmp": dict(k_list=[8, 6], seeds=[0]),
    }
    out = {}
    for name, kw in specs.items():
        spec = harness.default_spec(name)
        spec = dc_replace(spec, ell=10, max_iters=8, **kw)
        spec.twin = dc_replace(spec.twin, n=40, obs_grid_count=8, members=10)
        table = harness.run_experiment(spec)
        out[name] = [[harness._format_value(v) for v in row] for row in table.rows]
    with open(os.path.join(HERE, "harness_regen.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))


if __name__ == "__main__":
    if "--harness-only" in sys.argv:
        extract_harness_rows()
        regen_harness_rows()
        sys.exit(0)
    make_model_cases()
    make_problem_cases()
    extract_fixtures()
    extract_harness_rows()
    regen_harness_rows()
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
