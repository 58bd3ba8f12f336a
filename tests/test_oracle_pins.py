"""Pin the CPU oracle (oracle/) against the real reference.

The golden vectors in tests/golden were produced by importing the reference
itself (tests/golden/make_golden.py).  The LAPACK-free paths must match bit
for bit; LAPACK stages (Nystrom) to rounding.
"""

import json
import os

import numpy as np
import numpy.testing as npt
import pytest

from conftest import GOLDEN, unpack_problem
from oracle import l96
from oracle.algorithms import (NystromConfig, SolverConfig, make_lmp,
                               nystrom_evd, pcg, rhs_diff_sketch)
from oracle.obs import ObsNetwork
from oracle.twin import BASELINE_CONFIGS, TwinConfig, baseline_setup, build_setup


def test_tendencies_bit_exact(ref_model):
    g = ref_model
    npt.assert_array_equal(l96.tendency(g["x"], 8.0), g["tend"])
    npt.assert_array_equal(l96.tendency_tl(g["x"], g["v"]), g["tend_tl"])
    npt.assert_array_equal(l96.tendency_ad(g["x"], g["v"]), g["tend_ad"])


def test_integrate_tlm_adjoint_bit_exact(ref_model):
    g = ref_model
    traj = l96.integrate(g["x"], 0.025, 8, 8.0)
    npt.assert_array_equal(traj.states, g["int_states"])
    npt.assert_array_equal(traj.stages, g["int_stages"])
    npt.assert_array_equal(l96.tlm(traj, g["v"]), g["tlm"])
    npt.assert_array_equal(l96.adjoint(traj, g["adj_w"]), g["adj"])


def test_deterministic_truth_bit_exact(ref_model):
    npt.assert_array_equal(l96.deterministic_truth(40, 0.025, 8.0, 2000),
                           ref_model["truth40"])


def test_obs_with_time_zero(ref_model):
    g = ref_model
    traj = l96.Trajectory(g["obs0_states"], g["obs0_stages"], 0.025, 8.0)
    net = ObsNetwork([0, 3, 7], [0, 2, 4])
    npt.assert_array_equal(net.observe(traj), g["obs0_y"])
    npt.assert_array_equal(net.observe_tl(traj, g["v"][:10]), g["obs0_tl"])
    npt.assert_array_equal(net.observe_ad(traj, g["obs0_w"]), g["obs0_ad"])


def test_member_problem_bit_exact(ref_problem):
    g = ref_problem
    prob = unpack_problem(g, "tiny_")
    npt.assert_array_equal(prob.a_apply(g["tiny_z"]), g["tiny_az"])
    npt.assert_array_equal(prob.rhs(), g["tiny_rhs"])
    costs = [prob.quadratic_cost(g["tiny_z"][:, j]) for j in range(6)]
    npt.assert_array_equal(costs, g["tiny_cost"])
    npt.assert_array_equal(prob.a_apply(np.eye(40)), g["tiny_dense_a"])
    assert prob.n_matvecs == 2


def test_pcg_trace_bit_exact(ref_problem):
    g = ref_problem
    prob = unpack_problem(g, "tiny_")
    x, tr = pcg(prob.hessian_apply, prob.rhs(), SolverConfig(max_iters=8),
                cost_fn=prob.quadratic_cost)
    npt.assert_array_equal(tr.cost, g["tiny_pcg_cost"])
    npt.assert_array_equal(tr.resnorm, g["tiny_pcg_resnorm"])
    npt.assert_array_equal(x, g["tiny_pcg_x"])  # final increment (krylov.py:97)


def test_nystrom_lmp_pcg_match_reference(ref_problem):
    g = ref_problem
    prob = unpack_problem(g, "tiny_")
    approx = nystrom_evd(prob.a_apply, g["tiny_gamma"],
                         NystromConfig(ell=10, k=8, shift_mode="trace"))
    npt.assert_allclose(approx.values, g["tiny_nys_vals"], rtol=1e-12)
    assert approx.shift == float(g["tiny_nys_shift"])
    lmp = make_lmp(approx, "halfsum")
    assert lmp.theta == pytest.approx(float(g["tiny_theta"]), rel=1e-12)
    x, tr = pcg(prob.hessian_apply, prob.rhs(), SolverConfig(max_iters=8),
                precond=lmp, cost_fn=prob.quadratic_cost)
    npt.assert_allclose(tr.cost, g["tiny_lmp_cost"], rtol=1e-10)
    assert np.linalg.norm(x - g["tiny_lmp_x"]) <= 1e-10 * np.linalg.norm(g["tiny_lmp_x"])


@pytest.mark.parametrize("cfg_id,members,iters,k", [(1, (0, 4, 9), 30, 10), (2, (0, 17), 50, 20)])
def test_member_lmp_pcg_increments_match_reference(ref_problem, cfg_id, members, iters, k):
    """cfg1 / cfg2 member solves (Nystrom LMP from the control, own or shared
    trajectories) by the oracle against the reference's golden J traces and
    final increments x (rel 1e-10 at cfg1/2)."""
    g = ref_problem
    ctl = unpack_problem(g, f"cfg{cfg_id}_")
    gam = g[f"cfg{cfg_id}_gamma"]
    ell = gam.shape[1]
    lmp = make_lmp(nystrom_evd(ctl.a_apply, gam, NystromConfig(ell=ell, k=k, shift_mode="trace")),
                   "halfsum")
    st = baseline_setup(BASELINE_CONFIGS[1]) if cfg_id == 1 else None
    for j in members:
        m = st.members[j] if cfg_id == 1 else unpack_problem(g, f"cfg2_m{j}_")
        x, tr = pcg(m.hessian_apply, m.rhs(), SolverConfig(max_iters=iters), precond=lmp,
                    cost_fn=m.quadratic_cost)
        npt.assert_allclose(tr.cost, g[f"cfg{cfg_id}_m{j}_cost"], rtol=1e-10)
        xr = g[f"cfg{cfg_id}_m{j}_x"]
        assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr), (j, np.linalg.norm(x - xr))


def test_reference_harness_fixtures_regenerate():
    """The reference's own frontend fixtures (variant=none J traces of the
    harness, tiny.cfg / ensemble.cfg) regenerate exactly from the oracle
    twin builder: pins build_setup -> hessian_apply -> pcg -> cost."""
    with open(os.path.join(GOLDEN, "fixtures.json")) as fh:
        fx = json.load(fh)
    tw = TwinConfig(n=40, obs_grid_count=8, members=10)
    for key, vals in fx["control-lmp"].items():
        seed = int(key.split("/")[0])
        setup = build_setup(tw, trial_seed=seed)
        _, tr = pcg(setup.control.hessian_apply, setup.control.rhs(),
                    SolverConfig(max_iters=8), cost_fn=setup.control.quadratic_cost)
        assert [repr(c) for c in tr.cost] == vals
    setup = build_setup(tw, trial_seed=0)
    for key, vals in fx["ensemble-lmp"].items():
        m = setup.members[int(key.split("/")[1]) - 1]
        _, tr = pcg(m.hessian_apply, m.rhs(), SolverConfig(max_iters=8),
                    cost_fn=m.quadratic_cost)
        assert [repr(c) for c in tr.cost] == vals


def test_baseline_cfg1_builder_bit_exact(ref_problem):
    g = ref_problem
    st = baseline_setup(BASELINE_CONFIGS[1])
    npt.assert_array_equal(st.control.traj.states[0] - 0.0,
                           g["cfg1_states"][0])
    npt.assert_array_equal(st.control.traj.stages, g["cfg1_stages"])
    npt.assert_array_equal(st.control.innovation, g["cfg1_innov"])
    npt.assert_array_equal(st.ub.symbol, g["cfg1_symbol"])
    npt.assert_array_equal(np.stack([m.innovation for m in st.members]),
                           g["cfg1_member_innov"])
    npt.assert_array_equal(st.control.a_apply(g["cfg1_z"]), g["cfg1_az"])
    sk = rhs_diff_sketch(st.control, st.members)
    npt.assert_array_equal(sk.columns, g["cfg1_gamma"])
    approx = nystrom_evd(st.control.a_apply, sk, NystromConfig(10, 10, shift_mode="trace"))
    npt.assert_allclose(approx.values, g["cfg1_nys_vals"], rtol=1e-10)
    lmp = make_lmp(approx, "halfsum")
    for j in (0, 4, 9):
        m = st.members[j]
        _, tr = pcg(m.hessian_apply, m.rhs(), SolverConfig(max_iters=30),
                    precond=lmp, cost_fn=m.quadratic_cost)
        npt.assert_allclose(tr.cost, g[f"cfg1_m{j}_cost"], rtol=1e-10)


def test_baseline_cfg2_shift_path(ref_problem):
    """cfg2: ell=50 > n=40, the Gram matrix is singular and the reference
    succeeds on the first eps*trace(W) shift (SURVEY.md §7 hard part 2)."""
    g = ref_problem
    prob = unpack_problem(g, "cfg2_")
    for k in (10, 20, 50):
        approx = nystrom_evd(prob.a_apply, g["cfg2_gamma"],
                             NystromConfig(ell=50, k=k, shift_mode="trace"))
        assert approx.shift == float(g[f"cfg2_k{k}_shift"]) > 0.0
        assert approx.values.size == min(k, 40)
        ref = g[f"cfg2_k{k}_vals"]
        floor = 1e-10 * ref[0]
        big = ref >= 1e-6 * ref[0]
        npt.assert_allclose(approx.values[big], ref[big], rtol=1e-10)
        assert np.all(np.abs(approx.values[~big] - ref[~big]) <= floor)


def test_lanczos_matches_reference_fixture():
    """eig-sensitivity fixture (Lanczos over hessian_apply, diffusion B):
    oracle Lanczos on the oracle twin reproduces the reference's values."""
    import csv
    from oracle.algorithms import lanczos_eigs
    path = os.path.join(GOLDEN, "fixtures.json")
    with open(path) as fh:
        fx = json.load(fh)
    if "eig-sensitivity" not in fx:
        pytest.skip("fixture not extracted")
    tw = TwinConfig(n=40, obs_grid_count=8, members=10, cov_length=2.0)
    setup = build_setup(tw)
    vals, _ = lanczos_eigs(setup.control.hessian_apply, 40, min(40, tw.p + 80),
                           min(150, tw.p), seed=tw.seed)
    ref = [float(v) for v in fx["eig-sensitivity"]["D=2"]]
    npt.assert_allclose(vals[: len(ref)], ref, rtol=1e-10)
