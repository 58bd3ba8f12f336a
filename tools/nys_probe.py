"""cfg2/cfg1 Nystrom: Jacobi sweeps / shapes and the build_lmp time."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2605_23571_b200 import linalg, nystrom  # noqa: E402
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

orig = linalg.svd_jacobi


def spy(M, want_v=False):
    r = orig(M, want_v)
    print("   svd_jacobi cols x rows", tuple(M.shape), "want_v", want_v, "sweeps", linalg.last_svd_sweeps())
    return r


nystrom.svd_jacobi = spy
for c in (1, 2, 3):
    eng = EdaPass(build_ensemble(BASELINE_CONFIGS[c]))
    B = eng.rhs()
    print(f"cfg{c}")
    _, approx, _ = eng.build_lmp(B)
    v = approx.values
    print("   values", v[:3], v[-3:], "cond", v[0] / v[-1])
