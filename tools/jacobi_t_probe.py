"""Sweeps and time of the cluster Jacobi variants on the Nystrom T of a
config (CFG env, default 4): column tournament vs block tournament."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build, linalg, nystrom  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
eng = EdaPass(build_ensemble(cfg))
saved = []
orig = nystrom.svd_jacobi


def grab(M, want_v=False):
    saved.append(M.clone())
    return orig(M, want_v)


nystrom.svd_jacobi = grab
eng.build_lmp(eng.rhs())
nystrom.svd_jacobi = orig
T = saved[0]
want_v = T.shape[0] < 2 * 64 and cfg.n < cfg.ell  # the wide cfg2 route takes V
cols, rows = T.shape
ref = np.linalg.svd(T.cpu().numpy().T, compute_uv=False)
variants = os.environ.get("VARIANTS", "EDAK_JACOBI_BLOCK=1,EDAK_JACOBI_BLOCK=0").split(",")
for variant in variants:
    for k in ("EDAK_JACOBI_BLOCK", "EDAK_JACOBI_CLUSTER", "EDAK_JACOBI_SINGLE"):
        os.environ.pop(k, None)
    a, b = variant.split("=")
    os.environ[a] = b
    ts = []
    for _ in range(4):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        U, sig, _ = linalg.svd_jacobi(T, want_v=want_v)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    err = np.max(np.abs(sig.cpu().numpy() - ref) / ref[0])
    print(f"{cfg.name} T {rows}x{cols} {variant}: {np.median(ts):.3f} ms, "
          f"{linalg.last_svd_sweeps()} sweeps, max sigma err {err:.1e}")
