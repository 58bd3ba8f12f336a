"""Edge cases and error conventions the reference tests pin (SURVEY.md §8b:
ValueError for config / shape / theta problems, NystromBreakdownError, the
PCG RuntimeError messages), plus empty blocks through every C-ABI entry."""

from types import SimpleNamespace

import numpy as np
import pytest
import torch

from oracle import algorithms as oalg

# ------------------------------------------------------------ host logic --


def test_config_validation_matches_reference():
    from paper_2605_23571_b200.krylov import SolverConfig
    from paper_2605_23571_b200.nystrom import NystromConfig
    for bad in (dict(ell=5, k=0), dict(ell=5, k=6), dict(ell=5, k=3, q=0),
                dict(ell=5, k=3, shift_mode="bogus")):
        with pytest.raises(ValueError):
            NystromConfig(**bad)
        with pytest.raises(ValueError):  # the oracle restates the same checks
            oalg.NystromConfig(**bad)
    with pytest.raises(ValueError):
        SolverConfig(max_iters=0)
    assert NystromConfig(ell=5, k=5).q == 1


def test_theta_rules_and_lmp_validation():
    from paper_2605_23571_b200.lmp import SpectralLmp, choose_theta
    for rule in ("halfsum", "lambdak", "one"):
        for lam in (1.0, 1.5, 37.25):
            assert choose_theta(rule, lam) == oalg.choose_theta(rule, lam)
    with pytest.raises(ValueError, match="eigenvalues >= 1"):
        choose_theta("halfsum", 1.0 - 1e-7)
    assert choose_theta("halfsum", 1.0 - 1e-9) == pytest.approx(1.0)  # the 1e-8 slack
    with pytest.raises(ValueError, match="unknown theta rule"):
        choose_theta("median", 2.0)
    s = np.linalg.qr(np.random.default_rng(0).standard_normal((6, 2)))[0]
    with pytest.raises(ValueError):
        SpectralLmp(s, np.array([2.0, 1.0]), 0.0)
    with pytest.raises(ValueError):
        SpectralLmp(s, np.array([2.0, -1.0]), 1.0)
    SpectralLmp(s, np.array([2.0, -1e-13]), 1.0)  # rounding-level negatives pass


def test_network_factor_and_sketch_validation():
    from paper_2605_23571_b200.covariance import CirculantFactor, factor_taps
    from paper_2605_23571_b200.obs import ObsNetwork, position_maps
    from paper_2605_23571_b200.sketch import make_sketch
    with pytest.raises(ValueError, match="distinct"):
        ObsNetwork([0, 2, 2], [1])
    with pytest.raises(ValueError, match="distinct"):
        ObsNetwork([0, 2], [1, 1])
    with pytest.raises(ValueError, match="outside the ring"):
        position_maps(ObsNetwork([0, 40], [1]), 40, 8)
    with pytest.raises(ValueError, match="outside the window"):
        position_maps(ObsNetwork([0, 4], [9]), 40, 8)
    with pytest.raises(ValueError):
        CirculantFactor(40, np.ones(10))
    # a generator that does not decay needs more taps than the kernel takes
    n = 20000
    rng = np.random.default_rng(1)
    wide = CirculantFactor(n, 1.0 + rng.random(n // 2 + 1))
    with pytest.raises(ValueError, match="taps"):
        factor_taps(wide)
    setup = SimpleNamespace(members=[object()] * 3, cfg=SimpleNamespace(n=40))
    with pytest.raises(ValueError, match="ensemble size"):
        make_sketch("rhsdiff", setup, 4, np.random.default_rng(0))
    with pytest.raises(ValueError, match="unknown sketch kind"):
        make_sketch("sobol", setup, 3, np.random.default_rng(0))


def test_linearization_rejects_bad_stage_mode():
    from paper_2605_23571_b200.assim import Linearization
    with pytest.raises(ValueError, match="stage_mode"):
        Linearization(np.zeros((1, 3, 40)), 0.025, 8.0, None, None, None, stage_mode="cached")


# ------------------------------------------------------------------- GPU --


@pytest.fixture(scope="module")
def gpu():
    from paper_2605_23571_b200 import build
    build.build()


def _tiny_lin():
    from oracle import l96
    from oracle.cov import gaussian_factor
    from oracle.obs import ObsNetwork, strided_grid
    from paper_2605_23571_b200.assim import Linearization
    from paper_2605_23571_b200.covariance import CirculantFactor, DiagonalNoise
    x0 = 8.0 + np.random.default_rng(3).standard_normal(40)
    traj = l96.integrate(x0, 0.025, 8, 8.0)
    net = ObsNetwork(strided_grid(40, 20), list(range(1, 9)))
    ub = CirculantFactor(40, gaussian_factor(40, 0.8, 2.0).symbol)
    return Linearization(traj.states[None], 0.025, 8.0, net, ub, DiagonalNoise(1.0))


@pytest.mark.gpu
def test_empty_blocks_every_entry(gpu):
    """ncols = 0 is a no-op everywhere (returns EDAK_OK, writes nothing)."""
    from paper_2605_23571_b200 import _lib
    from paper_2605_23571_b200.linalg import gemm_nn, gemm_tn
    lin = _tiny_lin()
    dev = torch.device("cuda")
    Z = torch.empty((0, 40), dtype=torch.float64, device=dev)
    D = torch.empty((0, lin.p), dtype=torch.float64, device=dev)
    assert lin.hessian_cols(Z).shape == (0, 40)
    assert lin.hessian_cols(Z, ident=1.0).shape == (0, 40)
    assert lin.rhs_cols(D).shape == (0, 40)
    assert lin.cost_cols(Z, D).shape == (0,)
    assert lin.tl_cols(Z).shape == (0, lin.p)
    assert lin.ad_cols(D).shape == (0, 40)
    assert lin.dfac.apply_cols(Z).shape == (0, 40)
    S = torch.randn(3, 40, dtype=torch.float64, device=dev)
    assert gemm_tn(S, Z).numel() == 0
    null = None
    for fn, args in (
            ("edak_pcg_alpha", (40, 0, null, null, null, null, null, null, null, 1, null, null, 0, null)),
            ("edak_pcg_beta", (40, 0, null, null, null, null, 0.0, null, null, 9, null, null, 1, null)),
            ("edak_pcg_lmp_beta", (40, 3, 0, null, null, null, null, null, null, 0.0, null, null, 9,
                                   null, null, 1, null)),
            ("edak_lmp_apply", (40, 3, 0, null, null, null, null, null, null))):
        _lib.call(fn, *args)  # raises on a non-zero return code


@pytest.mark.gpu
def test_pcg_breakdown_messages(gpu):
    """krylov.py:73-74 / 82-84 messages on the device recurrence."""
    from paper_2605_23571_b200.krylov import SolverConfig, pcg
    rng = np.random.default_rng(4)
    a = rng.standard_normal((12, 12))
    spd = a @ a.T + 12 * np.eye(12)
    b = rng.standard_normal(12)
    with pytest.raises(RuntimeError, match="preconditioner is not positive definite"):
        pcg(lambda v: spd @ v, b, SolverConfig(max_iters=5), precond=lambda r: -r)
    with pytest.raises(RuntimeError, match=r"system matrix is not positive definite \(iteration 1\)"):
        pcg(lambda v: -spd @ v, b, SolverConfig(max_iters=5))
    x, tr = pcg(lambda v: spd @ v, b, SolverConfig(max_iters=40, residual_rtol=1e-10))
    assert tr.status == "converged" and np.allclose(spd @ x, b, atol=1e-8)
    ox, otr = oalg.pcg(lambda v: spd @ v, b, oalg.SolverConfig(max_iters=40, residual_rtol=1e-10))
    assert tr.iterations == otr.iterations


@pytest.mark.gpu
def test_nystrom_rejects_wrong_width(gpu):
    from paper_2605_23571_b200.nystrom import NystromConfig, nystrom_evd
    with pytest.raises(ValueError, match="columns"):
        nystrom_evd(lambda z: z, np.ones((10, 4)), NystromConfig(ell=5, k=3))
