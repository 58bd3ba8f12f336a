"""Time edak_chol_inv (fused blocked Cholesky + inverse) vs the unfused
potrf_shifted + trinv_upper at the Nystrom sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.linalg import chol_inv, potrf_shifted, trinv_upper  # noqa: E402


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1e3


rng = np.random.default_rng(0)
for l in (64, 128, 256):
    x = rng.standard_normal((l, l))
    W = torch.tensor((x @ x.T + l * np.eye(l)).T.copy(), device="cuda")
    a = t(lambda: chol_inv(W, 1))
    b = t(lambda: trinv_upper(potrf_shifted(W, 1)[0]))
    print(f"l={l}: chol_inv {a:.1f} us   potrf+trinv {b:.1f} us", flush=True)
