import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def ref_model():
    return dict(np.load(os.path.join(GOLDEN, "ref_model.npz")))


@pytest.fixture(scope="session")
def ref_problem():
    return dict(np.load(os.path.join(GOLDEN, "ref_problem.npz")))


def unpack_problem(g, prefix):
    """Rebuild an oracle MemberProblem from a golden dump (reference data)."""
    from oracle import l96
    from oracle.cov import CirculantFactor, DiagonalNoise
    from oracle.obs import ObsNetwork
    from oracle.problem import MemberProblem
    states, stages = g[prefix + "states"], g[prefix + "stages"]
    traj = l96.Trajectory(states, stages, 0.025, 8.0)
    net = ObsNetwork(g[prefix + "grid"], g[prefix + "times"])
    ub = CirculantFactor(states.shape[1], g[prefix + "symbol"])
    rn = DiagonalNoise(float(g[prefix + "sigma_obs"]))
    return MemberProblem(traj, net, ub, rn, g[prefix + "innov"])


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)
