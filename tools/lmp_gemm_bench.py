"""LMP GEMMs at the cfg4 group shape (n = 16384, k = 128, 100 members) and
the cfg5 shape (n = 262144, 128 members): edak_lmp_apply (W = S^T R, its
split-K reduction, z = R + S (c o W)) with the LMP-shaped kernels
(lmp_gemm.cu) vs the generic 64 x 64 / 64 x 112 tiles (EDAK_LMP_GEMM=0);
results against torch (fp64)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
lib = _lib.lib()
SHAPES = ((16384, 128, 100), (262144, 128, 128), (16384, 64, 50))
if os.environ.get("SHAPE"):
    SHAPES = (tuple(int(v) for v in os.environ["SHAPE"].split(",")),)
for n, k, M in SHAPES:
    g = torch.Generator(device="cuda").manual_seed(1)
    S = torch.linalg.qr(torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g))[0].t().contiguous()
    R = torch.randn(M, n, dtype=torch.float64, device="cuda", generator=g)
    coef = torch.rand(k, dtype=torch.float64, device="cuda", generator=g) - 0.9
    ref = R + ((R @ S.t()) * coef) @ S
    for flag in os.environ.get("FLAGS", "0,1").split(","):
        os.environ["EDAK_LMP_GEMM"] = flag
        work = torch.empty(int(lib.edak_lmp_work_doubles(n, k, M)), dtype=torch.float64, device="cuda")
        Z = torch.empty_like(R)
        f = lambda: _lib.call("edak_lmp_apply", n, k, M, S.data_ptr(), coef.data_ptr(), R.data_ptr(),
                              Z.data_ptr(), work.data_ptr(), _lib.stream())
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(20):
            f()
        e.record()
        torch.cuda.synchronize()
        us = s.elapsed_time(e) / 20 * 1e3
        err = float((Z - ref).norm() / ref.norm())
        tf = 4.0 * n * k * M / (us * 1e-6) / 1e12
        print(f"n={n} k={k} M={M} EDAK_LMP_GEMM={flag}: {us:.1f} us per apply ({tf:.1f} TFLOP/s), "
              f"rel err vs torch {err:.2e}", flush=True)

if os.environ.get("PROFILE"):
    # per-kernel device times (warm, back to back) via the CUDA profiler API
    from torch.profiler import ProfilerActivity, profile
    n, k, M = SHAPES[0]
    os.environ["EDAK_LMP_GEMM"] = os.environ.get("PROFILE")
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            f()
        torch.cuda.synchronize()
    for ev in prof.key_averages():
        if ev.device_type.name == "CUDA" or "k_" in ev.key:
            print(f"  {ev.key[:60]:60s} n={ev.count:3d} avg {ev.device_time_total / max(ev.count, 1):8.1f} us")
