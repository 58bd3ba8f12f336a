"""The fused LMP step of the batched PCG alone (edak_pcg_lmp_beta: W = S^T r
split-K, the partial reduction with r.Pr / beta, the p-update GEMM) at the
cfg4 member-group shape (n = 16384, k = 128, 100 members) and the cfg5
group (n = 262144, 256 members): device time per call (CUDA events over
REPS calls; inputs synthetic, statuses running)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
lib = _lib.lib()
reps = int(os.environ.get("REPS", "200"))
for n, k, M in ((16384, 128, 100), (262144, 128, 256)) if not os.environ.get("SHAPE") else (tuple(int(v) for v in os.environ["SHAPE"].split(",")),):
    g = torch.Generator(device="cuda").manual_seed(1)
    S = torch.linalg.qr(torch.randn(n, k, dtype=torch.float64, device="cuda", generator=g))[0].t().contiguous()
    R = torch.randn(M, n, dtype=torch.float64, device="cuda", generator=g)
    P = torch.randn(M, n, dtype=torch.float64, device="cuda", generator=g)
    coef = torch.rand(k, dtype=torch.float64, device="cuda", generator=g) - 0.9
    work = torch.ones(int(lib.edak_pcg_work_doubles(n, M)), dtype=torch.float64, device="cuda")
    lmpwork = torch.empty(int(lib.edak_lmp_work_doubles(n, k, M)), dtype=torch.float64, device="cuda")
    L = 4
    hist_rz = torch.ones(M, L, dtype=torch.float64, device="cuda")
    hist_J = torch.zeros(M, L, dtype=torch.float64, device="cuda")
    status = torch.zeros(M, dtype=torch.int32, device="cuda")
    iters = torch.zeros(M, dtype=torch.int32, device="cuda")

    def step():
        _lib.call("edak_pcg_lmp_beta", n, k, M, S.data_ptr(), coef.data_ptr(), R.data_ptr(), P.data_ptr(),
                  work.data_ptr(), lmpwork.data_ptr(), -1.0, hist_rz.data_ptr(), hist_J.data_ptr(), L,
                  status.data_ptr(), iters.data_ptr(), 1, _lib.stream())

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        step()
    e.record()
    torch.cuda.synchronize()
    print(f"n={n} k={k} M={M}: fused LMP step (S^T r + reduce/beta + p-update) "
          f"{1e3 * s.elapsed_time(e) / reps:.1f} us per call")
    if os.environ.get("PROFILE"):
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(50):
                step()
            torch.cuda.synchronize()
        for ev in sorted(prof.key_averages(), key=lambda v: -v.device_time_total):
            if ev.device_time_total > 0:
                print(f"   {ev.device_time_total / 50:8.1f} us  {ev.key[:70]}")
