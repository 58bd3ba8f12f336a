"""Time k_circ (U_B over a block) at cfg4/cfg5 shapes, with and without the
I + A epilogue (zadd + dot partials)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
if len(sys.argv) > 1:
    _lib._LIB = _lib.load(sys.argv[1])
from paper_2605_23571_b200.covariance import device_factor, gaussian_factor  # noqa: E402

for n, L, M in ((16384, 16.0, 200), (262144, 32.0, 256), (1024, 8.0, 50)):
    df = device_factor(gaussian_factor(n, 0.8, L))
    Z = torch.randn(M, n, dtype=torch.float64, device="cuda")
    out = torch.empty_like(Z)
    df.apply_cols(Z, out)
    ref = np.fft.irfft(np.fft.rfft(Z.cpu().numpy(), axis=1) * gaussian_factor(n, 0.8, L).symbol, n=n, axis=1)
    err = float(np.abs(out.cpu().numpy() - ref).max() / np.abs(ref).max())
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        df.apply_cols(Z, out)
    e.record()
    torch.cuda.synchronize()
    print(f"n={n} taps={df.ntaps} cols={M}: {s.elapsed_time(e) / 10 * 1e3:.1f} us  err {err:.1e}", flush=True)
