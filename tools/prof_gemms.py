"""Profiling driver: the cfg4 LMP GEMM shapes (S^T R, split-K reduce, and
the p-update S (c o W) + r + beta p) -- a few launches each, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
n, k, M = 16384, 128, int(os.environ.get("COLS", "100"))
dev = "cuda"
S = torch.randn(k, n, dtype=torch.float64, device=dev)
R = torch.randn(M, n, dtype=torch.float64, device=dev)
P = torch.randn(M, n, dtype=torch.float64, device=dev)
coef = torch.randn(k, dtype=torch.float64, device=dev)
beta = torch.randn(M, dtype=torch.float64, device=dev)
lib = _lib.lib()
W = torch.empty(M, k, dtype=torch.float64, device=dev)
part = torch.empty(int(lib.edak_lmp_work_doubles(n, k, M)), dtype=torch.float64, device=dev)
s = _lib.stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for it in range(6):
    ev[0].record()
    _lib.call("edak_gemm_tn", S.data_ptr(), n, R.data_ptr(), n, W.data_ptr(), k, k, M, n,
              part.data_ptr(), s)
    ev[1].record()
    _lib.call("edak_gemm_nn", S.data_ptr(), n, W.data_ptr(), k, coef.data_ptr(), R.data_ptr(), n,
              1.0, P.data_ptr(), n, n, M, k, s)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"tn+reduce {ev[0].elapsed_time(ev[1]) * 1e3:.1f} us  nn {ev[1].elapsed_time(ev[2]) * 1e3:.1f} us")
