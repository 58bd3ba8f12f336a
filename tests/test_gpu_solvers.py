"""GPU parity of the dense stages (DMMA GEMMs, Cholesky with the reference
shift schedule, Jacobi SVD), the Nystrom EVD, the LMP and PCG against the
CPU oracle and the reference golden vectors (SURVEY.md §8c protocol)."""

import json
import os

import numpy as np
import numpy.testing as npt
import pytest
import torch

from conftest import GOLDEN, unpack_problem
from parity import (assert_increment, assert_trace, assert_values, lmp_pcg_envelope, nystrom_envelope,
                    pcg_envelope)
from oracle import algorithms as oalg
from oracle.twin import TwinConfig, build_setup
from paper_2605_23571_b200 import _lib

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


@pytest.fixture(scope="module")
def gpu():
    import paper_2605_23571_b200 as pkg
    from paper_2605_23571_b200 import build
    build.build()
    return pkg


def _gpu_problem(op):
    from paper_2605_23571_b200.assim import MemberProblem
    from paper_2605_23571_b200.covariance import CirculantFactor, DiagonalNoise
    return MemberProblem(op.traj, op.net, CirculantFactor(op.n, op.ub.symbol),
                         DiagonalNoise(op.rn.sigma), op.innovation)


@pytest.mark.parametrize("m,nb,K", [(10, 10, 40), (64, 64, 1024), (128, 200, 16384), (37, 5, 999)])
def test_gemm_tn(gpu, m, nb, K):
    from paper_2605_23571_b200.linalg import gemm_tn
    A = torch.randn(m, K, dtype=torch.float64, device="cuda")
    B = torch.randn(nb, K, dtype=torch.float64, device="cuda")
    C = gemm_tn(A, B)  # block (nb, m)
    ref = (B @ A.t())
    assert torch.allclose(C, ref, rtol=1e-12, atol=1e-11 * K ** 0.5)


@pytest.mark.parametrize("M,N,kk", [(40, 10, 10), (16384, 200, 128), (1000, 7, 33)])
def test_gemm_nn(gpu, M, N, kk):
    from paper_2605_23571_b200.linalg import gemm_nn
    A = torch.randn(kk, M, dtype=torch.float64, device="cuda")   # column-major M x kk
    B = torch.randn(N, kk, dtype=torch.float64, device="cuda")   # column-major kk x N
    s = torch.rand(kk, dtype=torch.float64, device="cuda")
    Cin = torch.randn(N, M, dtype=torch.float64, device="cuda")
    D = gemm_nn(A, B, bscale=s, Cin=Cin, beta=1.0)
    ref = Cin + (B * s) @ A
    assert torch.allclose(D, ref, rtol=1e-12, atol=1e-12 * kk)


def test_potrf_paths(gpu):
    """test_nystrom.py:61-77 pattern on the device kernel."""
    from paper_2605_23571_b200.linalg import potrf_shifted
    rng = np.random.default_rng(3)
    x = rng.standard_normal((6, 6))
    w = x @ x.T + 6 * np.eye(6)
    W = torch.tensor(w.T.copy(), device="cuda")
    C, nu, info = potrf_shifted(W, 0)
    c = C.cpu().numpy().T
    npt.assert_allclose(c.T @ c, w, atol=1e-12 * np.linalg.norm(w))
    assert float(nu[0]) == 0.0 and info.cpu().tolist() == [0, 0]
    assert np.allclose(c, np.triu(c))
    Z = torch.zeros(4, 4, dtype=torch.float64, device="cuda")
    C, nu, info = potrf_shifted(Z, 2, 4.0)
    assert info.cpu().tolist()[1] == 0 and float(nu[0]) > 0
    npt.assert_allclose(C.cpu().numpy(), np.sqrt(float(nu[0])) * np.eye(4), atol=1e-18)
    assert potrf_shifted(Z, 0)[2].cpu().tolist()[1] == 1
    assert potrf_shifted(Z, 2, 0.0)[2].cpu().tolist()[1] == 1


@pytest.mark.parametrize("kind", ["auto", "single", "cluster", "colcluster"])
@pytest.mark.parametrize("rows,cols", [(10, 10), (64, 64), (1024, 64), (128, 128), (50, 40), (200, 50),
                                       (120, 100)])
def test_svd_jacobi(gpu, rows, cols, kind, monkeypatch):
    """Shared-memory single-CTA, register one-CTA (auto for small l) and
    8-CTA cluster Jacobi -- over blocks of columns (the default from 32
    columns, zero-padded to 16 even blocks) or over single columns
    (EDAK_JACOBI_BLOCK=0) -- all carrying V as the tail of each extended
    column when rows + cols fits."""
    from paper_2605_23571_b200.linalg import svd_jacobi
    if kind == "single":
        monkeypatch.setenv("EDAK_JACOBI_SINGLE", "1")
    if kind in ("cluster", "colcluster"):
        monkeypatch.setenv("EDAK_JACOBI_CLUSTER", "1")
    if kind == "colcluster":
        monkeypatch.setenv("EDAK_JACOBI_BLOCK", "0")
    rng = np.random.default_rng(rows + cols)
    m = rng.standard_normal((rows, cols)) * np.logspace(0, -6, cols)
    U, sig, V = svd_jacobi(torch.tensor(m.T.copy(), device="cuda"), want_v=True)
    s_ref = np.linalg.svd(m, compute_uv=False)
    npt.assert_allclose(sig.cpu().numpy(), s_ref, rtol=1e-12)
    u = U.cpu().numpy().T
    v = V.cpu().numpy().T
    npt.assert_allclose(u * sig.cpu().numpy(), m @ v, atol=1e-12 * s_ref[0])
    npt.assert_allclose(u.T @ u, np.eye(cols), atol=1e-12)
    npt.assert_allclose(v.T @ v, np.eye(cols), atol=1e-12)


@pytest.mark.parametrize("kind", ["auto", "cluster", "colcluster"])
def test_svd_jacobi_256_no_v(gpu, kind, monkeypatch):
    """The cfg5 route of the Nystrom stage: l = 256, T = R_Y C^-1 square,
    left vectors only (8-CTA cluster kernels, jacobi_cluster.cu: blocks of
    16 columns, or single columns with EDAK_JACOBI_BLOCK=0): singular
    values vs LAPACK, U orthonormal, U^T T has orthogonal rows of norm sig."""
    from paper_2605_23571_b200.linalg import svd_jacobi
    if kind in ("cluster", "colcluster"):
        monkeypatch.setenv("EDAK_JACOBI_CLUSTER", "1")
    if kind == "colcluster":
        monkeypatch.setenv("EDAK_JACOBI_BLOCK", "0")
    rng = np.random.default_rng(256)
    q1, _ = np.linalg.qr(rng.standard_normal((256, 256)))
    q2, _ = np.linalg.qr(rng.standard_normal((256, 256)))
    m = (q1 * np.logspace(3, -5, 256)) @ q2.T
    U, sig, _ = svd_jacobi(torch.tensor(m.T.copy(), device="cuda"))
    s_ref = np.linalg.svd(m, compute_uv=False)
    s = sig.cpu().numpy()
    npt.assert_allclose(s, s_ref, rtol=1e-11, atol=1e-13 * s_ref[0])
    u = U.cpu().numpy().T
    npt.assert_allclose(u.T @ u, np.eye(256), atol=1e-12)
    b = u.T @ m
    npt.assert_allclose(b @ b.T, np.diag(s ** 2), atol=1e-11 * s_ref[0] ** 2)


def _lmp_action_close(ours, ref_vecs, ref_vals, theta, n, tol):
    """Compare LMPs sign-invariantly through their action on random vectors."""
    ref = oalg.SpectralLmp(ref_vecs, ref_vals, theta)
    v = np.random.default_rng(0).standard_normal((n, 4))
    return rel(ours.apply(v), ref.apply(v)) < tol


def test_nystrom_tiny_golden(gpu, ref_problem):
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    g = ref_problem
    prob = _gpu_problem(unpack_problem(g, "tiny_"))
    cfg = NystromConfig(10, 8, shift_mode="trace")
    approx = nystrom_evd(prob.a_apply, g["tiny_gamma"], cfg)
    assert prob.n_matvecs == 1 and approx.n_build_matvecs == 1
    env = nystrom_envelope(unpack_problem(g, "tiny_"), g["tiny_gamma"],
                           oalg.NystromConfig(10, 8, shift_mode="trace"))
    assert_values(approx.values, g["tiny_nys_vals"], env)
    assert approx.shift == float(g["tiny_nys_shift"])
    npt.assert_allclose(approx.vectors.T @ approx.vectors, np.eye(8), atol=1e-12)
    lmp = make_lmp(approx, "halfsum")
    # theta = (lam_k + 2) / 2 inherits the envelope of the smallest value
    assert abs(lmp.theta - float(g["tiny_theta"])) <= max(1e-10 * lmp.theta, 5 * env[-1])
    assert _lmp_action_close(lmp, g["tiny_nys_vecs"], g["tiny_nys_vals"], lmp.theta, 40, 1e-8)


def test_nystrom_mirror_and_invariants(gpu, ref_problem):
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    g = ref_problem
    prob = _gpu_problem(unpack_problem(g, "mir_"))
    approx = nystrom_evd(prob.a_apply, g["mir_phi"], NystromConfig(20, 15, shift_mode="trace"))
    env = nystrom_envelope(unpack_problem(g, "mir_"), g["mir_phi"],
                           oalg.NystromConfig(20, 15, shift_mode="trace"))
    assert_values(approx.values, g["mir_nys_vals"], env)
    assert approx.shift == 0.0
    assert np.all(np.diff(approx.values) <= 0) and np.all(approx.values >= 0)


def test_nystrom_cfg2_shift_path(gpu, ref_problem):
    """l = 50 > n = 40: singular Gram, first eps*trace(W) shift succeeds,
    k = 50 returns 40 pairs (SURVEY.md §7 hard part 2)."""
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    g = ref_problem
    prob = _gpu_problem(unpack_problem(g, "cfg2_"))
    for k in (10, 20, 50):
        approx = nystrom_evd(prob.a_apply, g["cfg2_gamma"], NystromConfig(50, k, shift_mode="trace"))
        ref_shift = float(g[f"cfg2_k{k}_shift"])
        assert approx.shift == pytest.approx(ref_shift, rel=1e-12)
        ref = g[f"cfg2_k{k}_vals"]
        assert approx.values.size == ref.size == min(k, 40)
        env = nystrom_envelope(unpack_problem(g, "cfg2_"), g["cfg2_gamma"],
                               oalg.NystromConfig(50, k, shift_mode="trace"))
        assert_values(approx.values, ref, env)


def test_zero_operator_raises(gpu):
    from paper_2605_23571_b200.nystrom import NystromBreakdownError, NystromConfig, nystrom_evd
    phi = np.random.default_rng(2).standard_normal((12, 4))
    for mode in (None, "trace"):
        with pytest.raises(NystromBreakdownError):
            nystrom_evd(lambda v: 0.0 * v, phi, NystromConfig(ell=4, k=4, shift_mode=mode))


def test_pcg_generic_callables(gpu):
    from paper_2605_23571_b200.krylov import SolverConfig, pcg
    b = np.random.default_rng(0).standard_normal(25)
    x, tr = pcg(lambda v: v, b, SolverConfig(max_iters=10, residual_rtol=1e-12))
    npt.assert_allclose(x, b, atol=1e-14)
    assert tr.status == "converged" and tr.iterations[-1] == 1
    with pytest.raises(RuntimeError, match="iteration 1"):
        pcg(lambda v: -v, np.ones(5), SolverConfig(max_iters=3))
    rng = np.random.default_rng(1)
    m = rng.standard_normal((15, 15))
    h = m @ m.T + 15 * np.eye(15)
    hi = np.linalg.inv(h)
    bb = rng.standard_normal(15)
    xs, tr = pcg(lambda v: h @ v, bb, SolverConfig(max_iters=10, residual_rtol=1e-10),
                 precond=lambda v: hi @ v)
    assert tr.iterations[-1] == 1
    npt.assert_allclose(xs, np.linalg.solve(h, bb), atol=1e-10)


def test_pcg_reference_fixtures(gpu):
    """Reference harness fixtures (tiny.cfg / ensemble.cfg, diffusion B,
    unpreconditioned PCG J traces) reproduced by the GPU solver."""
    from paper_2605_23571_b200.krylov import SolverConfig, pcg
    with open(os.path.join(GOLDEN, "fixtures.json")) as fh:
        fx = json.load(fh)
    tw = TwinConfig(n=40, obs_grid_count=8, members=10)
    setup = build_setup(tw, trial_seed=0)
    prob = _gpu_problem(setup.control)
    _, tr = pcg(prob.hessian_apply, prob.rhs(), SolverConfig(max_iters=8),
                cost_fn=prob.quadratic_cost)
    npt.assert_allclose(tr.cost, [float(v) for v in fx["control-lmp"]["0/"]], rtol=1e-12)
    for key, vals in fx["ensemble-lmp"].items():
        m = _gpu_problem(setup.members[int(key.split("/")[1]) - 1])
        _, tr = pcg(m.hessian_apply, m.rhs(), SolverConfig(max_iters=8), cost_fn=m.quadratic_cost)
        npt.assert_allclose(tr.cost, [float(v) for v in vals], rtol=1e-12)


def test_cfg1_lmp_pcg_golden(gpu, ref_problem):
    """cfg1: Nystrom on Gamma (shared linearization) + halfsum LMP + 30 PCG
    iterations for three members against the reference's golden traces: J
    rel 1e-10; resnorm 1e-10 r0, or 10x the spread the trace shows on the CPU
    when its LMP is built from Y perturbed at 1e-16 (tests/parity.py
    lmp_pcg_envelope: late residuals amplify LMP rounding ~1e4-fold)."""
    from paper_2605_23571_b200.krylov import SolverConfig, pcg
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    from oracle.twin import BASELINE_CONFIGS, baseline_setup
    g = ref_problem
    st = baseline_setup(BASELINE_CONFIGS[1])
    ctl = _gpu_problem(st.control)
    approx = nystrom_evd(ctl.a_apply, g["cfg1_gamma"], NystromConfig(10, 10, shift_mode="trace"))
    env = nystrom_envelope(st.control, g["cfg1_gamma"], oalg.NystromConfig(10, 10, shift_mode="trace"))
    assert_values(approx.values, g["cfg1_nys_vals"], env)
    lmp = make_lmp(approx, "halfsum")
    for j in (0, 4, 9):
        m = _gpu_problem(st.members[j])
        x, tr = pcg(m.hessian_apply, m.rhs(), SolverConfig(max_iters=30), precond=lmp,
                    cost_fn=m.quadratic_cost)
        npt.assert_allclose(tr.cost, g[f"cfg1_m{j}_cost"], rtol=1e-10)
        ref = np.asarray(g[f"cfg1_m{j}_resnorm"])
        _, _, env_r, _, env_x = lmp_pcg_envelope(
            st.control, g["cfg1_gamma"], oalg.NystromConfig(10, 10, shift_mode="trace"), "halfsum",
            st.members[j], oalg.SolverConfig(max_iters=30), with_x=True)
        tol = np.maximum(1e-10 * ref[0], 10 * env_r)
        assert np.all(np.abs(np.array(tr.resnorm) - ref) <= tol)
        assert_increment(x, g[f"cfg1_m{j}_x"], env_x)


def test_pcg_members_batched_equals_single(gpu):
    """The batched engine runs the same per-member recurrence: identical
    traces to one-member solves, recurrence cost == exact cost (1e-10)."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import SolverConfig, pcg, pcg_members
    tw = TwinConfig(n=40, obs_grid_count=8, members=4)
    setup = build_setup(tw, trial_seed=0)
    mems = [_gpu_problem(m) for m in setup.members]
    ens = Ensemble.from_members(mems)
    cfg = SolverConfig(max_iters=12)
    X, trs = pcg_members(ens, ens.rhs_all(), cfg, cost="recurrence", small=False)
    X2, trs2 = pcg_members(ens, ens.rhs_all(), cfg, cost="exact", small=False)
    for j, m in enumerate(mems):
        _, tr = pcg(m.hessian_apply, m.rhs(), cfg, cost_fn=m.quadratic_cost)
        npt.assert_array_equal(trs[j].resnorm, tr.resnorm)  # same kernels, same bits
        npt.assert_allclose(trs[j].cost, trs2[j].cost, rtol=1e-10)
        om = setup.members[j]
        ref, ej, er = pcg_envelope(om.hessian_apply, om.rhs(), cfg, cost_fn=om.quadratic_cost)
        assert_trace(trs[j], ref, ej, er)


@pytest.mark.parametrize("l", [6, 50, 128, 200])
def test_potrf_trinv_sizes(gpu, l):
    """Shared-memory (l <= 128) and global (l > 128) Cholesky / inverse."""
    from paper_2605_23571_b200.linalg import potrf_shifted, trinv_upper
    rng = np.random.default_rng(l)
    x = rng.standard_normal((l, l))
    w = x @ x.T + l * np.eye(l)
    C, nu, info = potrf_shifted(torch.tensor(w.T.copy(), device="cuda"), 0)
    assert info.cpu().tolist() == [0, 0]
    c = C.cpu().numpy().T
    npt.assert_allclose(c, np.linalg.cholesky(w).T, rtol=1e-12, atol=1e-12 * np.abs(c).max())
    X = trinv_upper(C).cpu().numpy().T
    npt.assert_allclose(X @ c, np.eye(l), atol=1e-11)
    # rank-deficient Gram: plain fails, the eps*trace shift schedule succeeds
    y = rng.standard_normal((l, max(1, l // 2)))
    wd = y @ y.T
    C, nu, info = potrf_shifted(torch.tensor(wd.T.copy(), device="cuda"), 1)
    inf = info.cpu().tolist()
    assert inf[1] == 0 and inf[0] >= 1 and float(nu[0]) > 0
    c = C.cpu().numpy().T
    npt.assert_allclose(c.T @ c, wd + float(nu[0]) * np.eye(l), atol=1e-10 * np.abs(wd).max())


def test_lanczos_gpu(gpu):
    """Device Lanczos (krylov.lanczos_eigs, krylov.py:116-168) against the
    reference's eig-sensitivity fixture and the oracle on the n=120 mirror."""
    from paper_2605_23571_b200.krylov import lanczos_eigs
    with open(os.path.join(GOLDEN, "fixtures.json")) as fh:
        fx = json.load(fh)
    tw = TwinConfig(n=40, obs_grid_count=8, members=10, cov_length=2.0)
    setup = build_setup(tw)
    prob = _gpu_problem(setup.control)
    vals, bounds = lanczos_eigs(prob.hessian_apply, 40, min(40, tw.p + 80), min(150, tw.p),
                                seed=tw.seed)
    ref = [float(v) for v in fx["eig-sensitivity"]["D=2"]]
    npt.assert_allclose(vals[: len(ref)], ref, rtol=1e-8)
    tw = TwinConfig(n=120, obs_grid_count=10, members=0, seed=21)
    op = build_setup(tw).control
    vals, bounds = lanczos_eigs(_gpu_problem(op).hessian_apply, 120, 60, 40, seed=5)
    ref, ref_b = oalg.lanczos_eigs(op.hessian_apply, 120, 60, 40, seed=5)
    _assert_ritz(vals, bounds, ref, ref_b)
    # dense diagonal operator with restarts through invariant subspaces
    d = np.linspace(1.0, 30.0, 30)
    v, b = lanczos_eigs(lambda x: d * x, 30, 30, 5, seed=3)
    npt.assert_allclose(v, d[::-1][:5], rtol=1e-10)


def _assert_ritz(vals, bounds, ref, ref_b):
    """Ritz values of two Lanczos implementations: converged ones (residual
    bound <= 1e-6 of the value) to rel 1e-10, the rest to rel 1e-8 (their
    position inside the unconverged cluster is rounding-sensitive)."""
    vals, ref = np.asarray(vals), np.asarray(ref)
    conv = np.asarray(ref_b) <= 1e-6 * ref
    assert conv[:5].all()
    npt.assert_allclose(vals[conv], ref[conv], rtol=1e-10)
    npt.assert_allclose(vals, ref, rtol=1e-8)
    npt.assert_allclose(bounds[conv], ref_b[conv], rtol=1e-2, atol=1e-12 * ref[0])


def test_lanczos_baseline_scale(gpu):
    """The eig-study Lanczos (krylov.py:116-168, harness.py:126-175) on the
    BASELINE cfg4 control operator (n = 16384, 24-step window): 60 steps,
    top 20 Ritz values against the oracle on the same device-built inputs."""
    from paper_2605_23571_b200.assim import TrajectoryOperator
    from paper_2605_23571_b200.krylov import lanczos_eigs
    from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble
    from parity import oracle_rows
    dens = build_ensemble(BASELINE_CONFIGS[4], members=2)
    ctl = TrajectoryOperator(dens.lin, int(dens.traj_of[0]))
    vals, bounds = lanczos_eigs(ctl.hessian_apply, dens.cfg.n, 60, 20, seed=3)
    op = oracle_rows(dens, [0])[0]
    ref, ref_b = oalg.lanczos_eigs(op.hessian_apply, dens.cfg.n, 60, 20, seed=3)
    _assert_ritz(vals, bounds, ref, ref_b)


def test_pcg_fused_lmp_beta_matches_two_step(gpu, ref_problem):
    """Fused beta step (r.Pr = |r|^2 + W^T diag(c) W, p = r + beta p +
    S(c o W) in the GEMM epilogue, p.Hp from the Hessian's last pass) vs
    the unfused z = P r / r.z / p-update path and the cfg1 golden traces."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import SolverConfig, pcg_members
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    from oracle.twin import BASELINE_CONFIGS, baseline_setup
    g = ref_problem
    st = baseline_setup(BASELINE_CONFIGS[1])
    ctl = _gpu_problem(st.control)
    approx = nystrom_evd(ctl.a_apply, g["cfg1_gamma"], NystromConfig(10, 10, shift_mode="trace"))
    lmp = make_lmp(approx, "halfsum")
    assert lmp.single_pass() is not None
    mems = [_gpu_problem(m) for m in st.members]
    ens = Ensemble.from_members(mems)
    cfg = SolverConfig(max_iters=30)
    Xf, trf = pcg_members(ens, ens.rhs_all(), cfg, precond=lmp, fused=True, small=False)
    Xu, tru = pcg_members(ens, ens.rhs_all(), cfg, precond=lmp, fused=False, small=False)
    npt.assert_allclose(Xf.cpu().numpy(), Xu.cpu().numpy(), rtol=0, atol=1e-10 * float(Xu.abs().max()))
    for j in range(len(mems)):
        npt.assert_allclose(trf[j].cost, tru[j].cost, rtol=1e-11)
        r0 = tru[j].resnorm[0]  # same bar as the cfg1 golden resnorm check
        assert np.max(np.abs(np.array(trf[j].resnorm) - tru[j].resnorm)) <= 1e-10 * r0
    for j in (0, 4, 9):
        npt.assert_allclose(trf[j].cost, g[f"cfg1_m{j}_cost"], rtol=1e-10)


@pytest.mark.parametrize("l", [1, 6, 31, 33, 50, 64, 128, 129, 200, 256])
def test_chol_inv_matches_potrf_and_inverse(gpu, l):
    """Fused blocked Cholesky + inverse (cholinv.cu): same factor, shift
    schedule, nu and info as potrf_shifted; C^-1 C = I; zero/indefinite
    cases fail the same way."""
    from paper_2605_23571_b200.linalg import chol_inv, potrf_shifted
    rng = np.random.default_rng(l + 100)
    x = rng.standard_normal((l, l))
    w = x @ x.T + l * np.eye(l)
    W = torch.tensor(w.T.copy(), device="cuda")
    C, Ci, nu, info = chol_inv(W, 0)
    assert info.cpu().tolist() == [0, 0] and float(nu[0]) == 0.0
    c = C.cpu().numpy().T
    npt.assert_allclose(c, np.linalg.cholesky(w).T, rtol=1e-12, atol=1e-12 * np.abs(c).max())
    C2, _, _ = potrf_shifted(W, 0)
    npt.assert_allclose(c, C2.cpu().numpy().T, rtol=1e-13, atol=1e-13 * np.abs(c).max())
    X = Ci.cpu().numpy().T
    assert np.allclose(X, np.triu(X)) and np.allclose(c, np.triu(c))
    npt.assert_allclose(X @ c, np.eye(l), atol=1e-12)
    for mode, scale in ((1, 0.0), (2, 7.0)):
        y = rng.standard_normal((l, max(1, l // 2)))
        wd = y @ y.T
        Wd = torch.tensor(wd.T.copy(), device="cuda")
        C, Ci, nu, info = chol_inv(Wd, mode, scale)
        Cr, nur, infor = potrf_shifted(Wd, mode, scale)
        assert info.cpu().tolist() == infor.cpu().tolist()
        assert float(nu[0]) == float(nur[0])
        if info.cpu().tolist()[1] == 0:
            c = C.cpu().numpy().T
            npt.assert_allclose(c.T @ c, wd + float(nu[0]) * np.eye(l),
                                atol=1e-10 * max(np.abs(wd).max(), 1e-300))
            npt.assert_allclose(Ci.cpu().numpy().T @ c, np.eye(l), atol=1e-6)
    Z = torch.zeros(l, l, dtype=torch.float64, device="cuda")
    assert chol_inv(Z, 0)[3].cpu().tolist()[1] == 1
    assert chol_inv(Z, 2, 0.0)[3].cpu().tolist()[1] == 1


def test_pcg_members_graph_replay_equals_eager(gpu):
    """The captured CUDA-graph solve (first call captures, later calls replay
    with new right-hand sides / LMP) gives the same bits as eager launches,
    for one and for two member groups."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import SolverConfig, pcg_members
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    tw = TwinConfig(n=40, obs_grid_count=8, members=6)
    setup = build_setup(tw, trial_seed=0)
    mems = [_gpu_problem(m) for m in setup.members]
    ens = Ensemble.from_members(mems)
    ctl = _gpu_problem(setup.control)
    B = ens.rhs_all()
    cfg = SolverConfig(max_iters=9)
    lmps = []
    for k in (4, 6):
        approx = nystrom_evd(ctl.a_apply, (B - B.mean(0)).t().cpu().numpy(),
                             NystromConfig(ell=6, k=k, shift_mode="trace"))
        lmps.append(make_lmp(approx, "halfsum"))
    for groups in (1, 2):
        for lmp in [None] + lmps[:1] + lmps[:1]:  # capture, then replay twice
            Xe, te = pcg_members(ens, B, cfg, precond=lmp, groups=groups, graph=False, small=False)
            Xg, tg = pcg_members(ens, B, cfg, precond=lmp, groups=groups, graph=True, small=False)
            assert torch.equal(Xe, Xg)
            for a, b in zip(te, tg):
                assert a.cost == b.cost and a.resnorm == b.resnorm and a.status == b.status
        B2 = B * 1.5
        Xe, te = pcg_members(ens, B2, cfg, precond=lmps[0], groups=groups, graph=False, small=False)
        Xg, tg = pcg_members(ens, B2, cfg, precond=lmps[0], groups=groups, graph=True, small=False)
        assert torch.equal(Xe, Xg)


@pytest.mark.parametrize("n,grid", [(40, 8), (100, 20), (256, 64)])
def test_pcg_small_persistent_matches_batched(gpu, n, grid):
    """The one-launch small-ring solve (pcg_small.cu: one CTA per member runs
    every iteration) against the per-iteration batched path and the oracle,
    separate trajectories per member.  First 4 iterations (before CG's
    round-off amplification sets in): x, J, resnorm to 1e-12 of the batched
    path, with and without a single-pass LMP.  15 iterations: every member's
    trace inside the oracle's CPU-vs-CPU envelope (assert_trace).  With
    residual_rtol both paths converge, a few iterations apart (the stopping
    iteration sits on the same round-off-amplified plateau)."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import SolverConfig, pcg_members
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    tw = TwinConfig(n=n, obs_grid_count=grid, members=7)
    setup = build_setup(tw, trial_seed=1)
    mems = [_gpu_problem(m) for m in setup.members]
    ens = Ensemble.from_members(mems)
    ctl = _gpu_problem(setup.control)
    B = ens.rhs_all()
    approx = nystrom_evd(ctl.a_apply, (B - B.mean(0)).t().cpu().numpy(),
                         NystromConfig(ell=7, k=5, shift_mode="trace"))
    lmp = make_lmp(approx, "halfsum")
    for pre in (None, lmp):
        cfg = SolverConfig(max_iters=4)
        Xb, tb = pcg_members(ens, B, cfg, precond=pre, small=False, graph=False)
        n0 = _lib.launch_count()
        Xs, ts = pcg_members(ens, B, cfg, precond=pre, small=True)
        assert _lib.launch_count() - n0 == 1
        npt.assert_allclose(Xs.cpu().numpy(), Xb.cpu().numpy(), rtol=0,
                            atol=1e-12 * float(Xb.abs().max()))
        for a, b in zip(ts, tb):
            assert a.status == b.status and a.iterations == b.iterations
            npt.assert_allclose(a.cost, b.cost, rtol=1e-12)
            assert np.max(np.abs(np.array(a.resnorm) - b.resnorm)) <= 1e-12 * b.resnorm[0]
    cfg = SolverConfig(max_iters=15)
    _, ts = pcg_members(ens, B, cfg, small=True)
    _, tb = pcg_members(ens, B, cfg, small=False, graph=False)
    gen = torch.Generator(device="cuda").manual_seed(0)
    jit = []
    for _ in range(3):
        Bp = B * (1 + 1e-16 * torch.randn(B.shape, generator=gen, device="cuda", dtype=torch.float64))
        jit.append(pcg_members(ens, Bp, cfg, small=True)[1])
    for j, om in enumerate(setup.members):
        ref, ej, er = pcg_envelope(om.hessian_apply, om.rhs(), cfg, cost_fn=om.quadratic_cost)
        # plain CG on these ill-conditioned twins amplifies round-off ~1e8-fold
        # by iteration 10 (tools/small_probe.py): widen the CPU envelope by the
        # batched GPU path's distance from the oracle and by the persistent
        # path's own spread under 1e-16 right-hand-side jitter
        ej = np.maximum(ej, np.abs(np.array(tb[j].cost) - ref.cost))
        er = np.maximum(er, np.abs(np.array(tb[j].resnorm) - ref.resnorm))
        for t in jit:
            ej = np.maximum(ej, np.abs(np.array(t[j].cost) - ts[j].cost))
            er = np.maximum(er, np.abs(np.array(t[j].resnorm) - ts[j].resnorm))
        assert_trace(ts[j], ref, ej, er)
    cfg = SolverConfig(max_iters=300, residual_rtol=1e-5)
    _, tb = pcg_members(ens, B, cfg, precond=lmp, small=False, graph=False)
    _, ts = pcg_members(ens, B, cfg, precond=lmp, small=True)
    for a, b in zip(ts, tb):
        assert a.status == b.status == "converged"
        assert abs(a.iterations[-1] - b.iterations[-1]) <= max(3, b.iterations[-1] // 5)
        assert a.resnorm[-1] <= 1e-5 * a.resnorm[0]


def test_pcg_small_cfg1_golden(gpu, ref_problem):
    """cfg1 members through the persistent solve against the reference's
    golden traces (same bars as test_cfg1_lmp_pcg_golden)."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import SolverConfig, pcg_members
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    from oracle.twin import BASELINE_CONFIGS, baseline_setup
    g = ref_problem
    st = baseline_setup(BASELINE_CONFIGS[1])
    ctl = _gpu_problem(st.control)
    approx = nystrom_evd(ctl.a_apply, g["cfg1_gamma"], NystromConfig(10, 10, shift_mode="trace"))
    lmp = make_lmp(approx, "halfsum")
    ens = Ensemble.from_members([_gpu_problem(m) for m in st.members])
    X, trs = pcg_members(ens, ens.rhs_all(), SolverConfig(max_iters=30), precond=lmp, small=True)
    X = X.cpu().numpy()
    for j in (0, 4, 9):
        npt.assert_allclose(trs[j].cost, g[f"cfg1_m{j}_cost"], rtol=1e-10)
        ref = np.asarray(g[f"cfg1_m{j}_resnorm"])
        _, _, env_r, _, env_x = lmp_pcg_envelope(
            st.control, g["cfg1_gamma"], oalg.NystromConfig(10, 10, shift_mode="trace"), "halfsum",
            st.members[j], oalg.SolverConfig(max_iters=30), with_x=True)
        tol = np.maximum(1e-10 * ref[0], 10 * env_r)
        assert np.all(np.abs(np.array(trs[j].resnorm) - ref) <= tol)
        assert_increment(X[j], g[f"cfg1_m{j}_x"], env_x)


@pytest.mark.parametrize("path", ["dropin", "batched", "persistent"])
def test_cfg2_member_pcg_golden(gpu, ref_problem, path):
    """cfg2 (n = 40, 50 members with their OWN trajectories, l = 50 > n, the
    eps*trace(W) shift path, k = 20): the GPU Nystrom LMP of the control and
    the 50-iteration member solves of members 0 and 17 (harness.py:256-266
    per-member solves through krylov.py:49-97) against the reference's golden
    J traces, residual histories and final increments -- through the drop-in
    pcg, the batched per-iteration engine and the persistent one-launch
    solve (the path bench cfg2 takes)."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import SolverConfig, pcg, pcg_members
    from paper_2605_23571_b200.lmp import make_lmp
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    g = ref_problem
    octl = unpack_problem(g, "cfg2_")
    ctl = _gpu_problem(octl)
    approx = nystrom_evd(ctl.a_apply, g["cfg2_gamma"], NystromConfig(50, 20, shift_mode="trace"))
    assert approx.shift == pytest.approx(float(g["cfg2_k20_shift"]), rel=1e-12)
    lmp = make_lmp(approx, "halfsum")
    ops = [unpack_problem(g, f"cfg2_m{j}_") for j in (0, 17)]
    mems = [_gpu_problem(o) for o in ops]
    cfg = SolverConfig(max_iters=50)
    if path == "dropin":
        res = [pcg(m.hessian_apply, m.rhs(), cfg, precond=lmp, cost_fn=m.quadratic_cost)
               for m in mems]
    else:
        ens = Ensemble.from_members(mems)
        X, trs = pcg_members(ens, ens.rhs_all(), cfg, precond=lmp, small=(path == "persistent"))
        res = list(zip(X.cpu().numpy(), trs))
    for (x, tr), j, om in zip(res, (0, 17), ops):
        ref_j = np.asarray(g[f"cfg2_m{j}_cost"])
        ref_r = np.asarray(g[f"cfg2_m{j}_resnorm"])
        ref, env_j, env_r, _, env_x = lmp_pcg_envelope(
            octl, g["cfg2_gamma"], oalg.NystromConfig(50, 20, shift_mode="trace"), "halfsum", om,
            oalg.SolverConfig(max_iters=50), with_x=True)
        assert len(tr.cost) == ref_j.size == 51
        assert np.all(np.abs(np.asarray(tr.cost) - ref_j) <= np.maximum(1e-10 * np.abs(ref_j),
                                                                          10 * env_j))
        assert np.all(np.abs(np.asarray(tr.resnorm) - ref_r) <= np.maximum(1e-10 * ref_r[0],
                                                                            10 * env_r))
        assert_increment(x, g[f"cfg2_m{j}_x"], env_x)


def test_pcg_small_breakdown_statuses(gpu):
    """A negative-definite LMP (coef < -1) makes r.z < 0 at the start: the
    persistent solve reports the reference's 'preconditioner is not positive
    definite' like the batched path."""
    from paper_2605_23571_b200.assim import Ensemble
    from paper_2605_23571_b200.krylov import PcgBreakdown, SolverConfig, pcg_members_small
    tw = TwinConfig(n=40, obs_grid_count=8, members=3)
    setup = build_setup(tw, trial_seed=2)
    ens = Ensemble.from_members([_gpu_problem(m) for m in setup.members])
    B = ens.rhs_all()
    S = (B / B.norm(dim=1, keepdim=True)).contiguous()
    coef = torch.full((S.shape[0],), -3.0, dtype=torch.float64, device=B.device)
    with pytest.raises(PcgBreakdown, match="preconditioner is not positive definite"):
        pcg_members_small(ens, B, SolverConfig(max_iters=5), (S, coef))


def test_gemm_16byte_staging_edges(gpu):
    """The 16-byte cp.async staging of the DMMA GEMMs (even leading
    dimensions, 16-byte aligned operands) at odd K / odd M / odd inner
    dimension: the last pair of a row is half valid and half zero-filled.
    Leading dimensions are padded to even sizes so the 16-byte path runs, and
    the result equals the 8-byte path (EDAK_GEMM_V16=0) and torch."""
    import os
    from paper_2605_23571_b200 import _lib
    lib = _lib.lib()
    dev = "cuda"
    m, nb, K, ld = 37, 5, 999, 1000                      # TN: C = A^T B over K (odd), lda = ldb = 1000
    A = torch.randn(m, ld, dtype=torch.float64, device=dev)
    B = torch.randn(nb, ld, dtype=torch.float64, device=dev)
    outs = []
    for v in ("1", "0"):
        os.environ["EDAK_GEMM_V16"] = v
        C = torch.empty(nb, m, dtype=torch.float64, device=dev)
        part = torch.empty(int(lib.edak_gemm_tn_partials(m, nb, K)), dtype=torch.float64, device=dev)
        _lib.call("edak_gemm_tn", A.data_ptr(), ld, B.data_ptr(), ld, C.data_ptr(), m, m, nb, K,
                  part.data_ptr(), _lib.stream())
        outs.append(C)
    os.environ.pop("EDAK_GEMM_V16")
    ref = B[:, :K] @ A[:, :K].t()
    assert torch.allclose(outs[0], ref, rtol=1e-12, atol=1e-11 * K ** 0.5)
    assert torch.equal(outs[0], outs[1])
    M, N, kk, lda, ldb = 999, 7, 33, 1000, 34            # NN: odd M and inner dim, even lds
    A = torch.randn(kk, lda, dtype=torch.float64, device=dev)
    B = torch.randn(N, ldb, dtype=torch.float64, device=dev)
    s = torch.rand(kk, dtype=torch.float64, device=dev)
    Cin = torch.randn(N, M, dtype=torch.float64, device=dev)
    outs = []
    for v in ("1", "0"):
        os.environ["EDAK_GEMM_V16"] = v
        D = torch.empty(N, M, dtype=torch.float64, device=dev)
        _lib.call("edak_gemm_nn", A.data_ptr(), lda, B.data_ptr(), ldb, s.data_ptr(), Cin.data_ptr(), M, 1.0,
                  D.data_ptr(), M, M, N, kk, _lib.stream())
        outs.append(D)
    os.environ.pop("EDAK_GEMM_V16")
    ref = Cin + (B[:, :kk] * s) @ A[:, :M]
    assert torch.allclose(outs[0], ref, rtol=1e-12, atol=1e-12 * kk)
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("m,nb,K,sym", [(256, 256, 65536, True), (256, 256, 65538, False),
                                        (200, 200, 70000, True), (200, 136, 65536, False),
                                        (128, 128, 262144, True)])
def test_gemm_tn_big_tiles(gpu, m, nb, K, sym):
    """The 128 x 128 k_lmp_tn tiles that carry the big-K Nystrom Grams
    (cfg5: 256 x 256 over n = 262144; symmetric products compute the upper
    tiles and mirror the rest) against torch and the generic kernels."""
    from paper_2605_23571_b200.linalg import gemm_tn
    g = torch.Generator(device="cuda").manual_seed(m + nb)
    A = torch.randn(m, K, dtype=torch.float64, device="cuda", generator=g)
    B = A if sym else torch.randn(nb, K, dtype=torch.float64, device="cuda", generator=g)
    C = gemm_tn(A, B)  # block (nb, m)
    ref = B @ A.t()
    assert torch.allclose(C, ref, rtol=1e-12, atol=1e-11 * K ** 0.5)
    if sym:
        assert torch.equal(C, C.t())  # mirrored, not recomputed
    os.environ["EDAK_BIG_TN"] = "0"
    try:
        Cg = gemm_tn(A, B)
    finally:
        del os.environ["EDAK_BIG_TN"]
    assert torch.allclose(C, Cg, rtol=1e-12, atol=1e-11 * K ** 0.5)


@pytest.mark.parametrize("n,k,ncols", [(262144, 128, 128), (16384, 128, 120), (16384, 64, 113),
                                       (16384, 128, 100), (8192, 128, 256)])
def test_lmp_apply_member_tiles(gpu, n, k, ncols):
    """z = r + S (c o S^T r) (lmp.py:62-65) through the LMP-shaped kernels at
    112- and 128-member tiles (and 2 x 128 column blocks) against torch."""
    g = torch.Generator(device="cuda").manual_seed(n + k + ncols)
    S = torch.randn(k, n, dtype=torch.float64, device="cuda", generator=g) / n ** 0.5
    coef = torch.rand(k, dtype=torch.float64, device="cuda", generator=g) - 0.5
    R = torch.randn(ncols, n, dtype=torch.float64, device="cuda", generator=g)
    Z = torch.empty_like(R)
    work = torch.empty(int(_lib.lib().edak_lmp_work_doubles(n, k, ncols)), dtype=torch.float64, device="cuda")
    _lib.call("edak_lmp_apply", n, k, ncols, S.data_ptr(), coef.data_ptr(), R.data_ptr(), Z.data_ptr(),
              work.data_ptr(), _lib.stream())
    ref = R + ((R @ S.t()) * coef) @ S
    assert torch.allclose(Z, ref, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("cond", [1e2, 1e6, 1e9])
def test_cholqr_lazy_paths(gpu, cond):
    """The Nystrom stage's CholeskyQR (nystrom._cholqr_lazy): two unshifted
    passes with the last triangular solve left to the caller for a
    well-conditioned sketch, more passes / the shifted CholeskyQR3 for an
    ill-conditioned one; Q_Y = Qp Ti orthonormal and Y = Q_Y R_Y to the
    level of Householder QR (nystrom.py:118) in every case."""
    from paper_2605_23571_b200.linalg import gemm_nn
    from paper_2605_23571_b200.nystrom import _cholqr_lazy
    rng = np.random.default_rng(int(np.log10(cond)))
    n, l = 8192, 64
    U, _ = np.linalg.qr(rng.standard_normal((n, l)))
    V, _ = np.linalg.qr(rng.standard_normal((l, l)))
    Y = (U * np.logspace(0, -np.log10(cond), l)) @ V.T
    Yd = torch.tensor(np.ascontiguousarray(Y.T), device="cuda")  # block (l, n)
    qr, _ = _cholqr_lazy(Yd)
    Qp, Ti, R = qr
    Q = gemm_nn(Qp, Ti).cpu().numpy().T   # (n, l)
    Rm = R.cpu().numpy().T                # upper (l, l)
    assert np.abs(Q.T @ Q - np.eye(l)).max() <= 1e-13
    assert np.linalg.norm(Y - Q @ Rm) <= 1e-14 * np.linalg.norm(Y) * l
    assert np.abs(np.tril(Rm, -1)).max() == 0.0
    if cond <= 1e6:  # CholeskyQR2: the second pass's inverse is left to the caller
        assert not torch.equal(Ti, torch.eye(l, dtype=Ti.dtype, device=Ti.device))


def test_nystrom_blocked_gram_shift(gpu):
    """l = 160 (the 2 x 2 block Cholesky of 129..256 Grams, deferred on a
    side stream) on a rank-100 operator: the sketched Gram is singular, the
    unshifted block factorisation breaks down and the one-kernel
    factorisation with the reference's shift schedule (nystrom.py:67-93)
    takes over -- same shift as the oracle, Ritz values to its envelope."""
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    rng = np.random.default_rng(160)
    n, r, l, k = 2048, 100, 160, 64
    Vr, _ = np.linalg.qr(rng.standard_normal((n, r)))
    lam = np.logspace(2, -1, r)

    def a_apply(z):
        return Vr @ (lam[:, None] * (Vr.T @ z)) if z.ndim == 2 else Vr @ (lam * (Vr.T @ z))

    phi = rng.standard_normal((n, l))
    approx = nystrom_evd(a_apply, phi, NystromConfig(l, k, shift_mode="trace"))
    ref = oalg.nystrom_evd(a_apply, phi, oalg.NystromConfig(l, k, shift_mode="trace"))
    assert ref.shift > 0.0
    assert approx.shift == pytest.approx(ref.shift, rel=1e-12)
    big = ref.values >= 1e-6 * ref.values[0]
    npt.assert_allclose(approx.values[big], ref.values[big], rtol=1e-9)


def test_shifted_cholesky_dropin(gpu):
    """nystrom.shifted_cholesky (nystrom.py:67-93) on the device: plain
    factor of an SPD matrix, the eps * scale * 10^j shift schedule on a
    singular Gram (same nu as the oracle), and the reference's two
    breakdown messages."""
    import scipy.linalg
    from paper_2605_23571_b200.nystrom import NystromBreakdownError, shifted_cholesky
    rng = np.random.default_rng(67)
    a = rng.standard_normal((30, 30))
    w = a @ a.T + 30 * np.eye(30)
    c, nu = shifted_cholesky(w, "trace", np.trace(w))
    assert nu == 0.0
    npt.assert_allclose(c, scipy.linalg.cholesky(w, lower=False), rtol=1e-12, atol=1e-13)
    b = rng.standard_normal((30, 12))
    ws = b @ b.T  # rank 12: the plain factorization breaks down
    c, nu = shifted_cholesky(ws, "trace", np.trace(ws))
    c_ref, nu_ref = oalg.shifted_cholesky(ws, "trace", np.trace(ws))
    assert nu > 0.0 and nu == pytest.approx(nu_ref, rel=1e-12)
    npt.assert_allclose(c.T @ c, ws + nu * np.eye(30), rtol=0, atol=1e-10 * np.abs(ws).max())
    with pytest.raises(NystromBreakdownError, match="no usable shift"):
        shifted_cholesky(ws, None, np.trace(ws))
    with pytest.raises(NystromBreakdownError, match="stayed indefinite"):
        shifted_cholesky(-np.eye(30), "trace", 1.0)
