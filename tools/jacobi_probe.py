"""Sweeps and time of the device Jacobi SVD on random / Nystrom-like T."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
lib = _lib.lib()


def run(Mnp):
    M = torch.from_numpy(np.ascontiguousarray(Mnp)).cuda()
    cols, rows = M.shape
    U = torch.empty_like(M)
    sig = torch.empty(cols, dtype=torch.float64, device="cuda")
    work = torch.empty(int(lib.edak_svd_work_doubles(rows, cols)), dtype=torch.float64, device="cuda")
    for _ in range(2):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.call("edak_svd_jacobi", M.data_ptr(), rows, cols, U.data_ptr(), sig.data_ptr(), None,
                  work.data_ptr(), _lib.stream())
        e.record()
        torch.cuda.synchronize()
    ref = np.linalg.svd(Mnp.T, compute_uv=False)
    err = np.max(np.abs(sig.cpu().numpy() - ref) / ref[0])
    return s.elapsed_time(e), int(work[-1].item()), err


rng = np.random.default_rng(0)
for l in (64, 128, 256):
    A = rng.standard_normal((l, l))
    t, sw, err = run(A)
    print(f"random {l}: {t:.3f} ms, {sw} sweeps, err {err:.1e}")
    Q, _ = np.linalg.qr(rng.standard_normal((l, l)))
    d = np.logspace(0, -8, l)
    A = (Q * d) @ np.linalg.qr(rng.standard_normal((l, l)))[0]
    t, sw, err = run(np.triu(A))
    print(f"graded-triu {l}: {t:.3f} ms, {sw} sweeps, err {err:.1e}")


def run_v(rows, cols, single):
    os.environ["EDAK_JACOBI_SINGLE"] = "1" if single else ""
    if not single:
        del os.environ["EDAK_JACOBI_SINGLE"]
    m = rng.standard_normal((rows, cols)) * np.logspace(0, -6, cols)
    M = torch.from_numpy(np.ascontiguousarray(m.T)).cuda()
    U = torch.empty_like(M)
    V = torch.empty(cols, cols, dtype=torch.float64, device="cuda")
    sig = torch.empty(cols, dtype=torch.float64, device="cuda")
    work = torch.empty(int(lib.edak_svd_work_doubles(rows, cols)), dtype=torch.float64, device="cuda")
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.call("edak_svd_jacobi", M.data_ptr(), rows, cols, U.data_ptr(), sig.data_ptr(), V.data_ptr(),
                  work.data_ptr(), _lib.stream())
        e.record()
        torch.cuda.synchronize()
    kind = "single" if single else ("cluster" if os.environ.get("EDAK_JACOBI_CLUSTER") else "auto")
    print(f"want_v {rows}x{cols} {kind}: {s.elapsed_time(e):.3f} ms, "
          f"{int(work[-1].item())} sweeps")


for rows, cols in ((50, 40), (40, 10), (64, 64), (128, 128), (200, 50)):
    for single in (True, False):
        run_v(rows, cols, single)
    os.environ["EDAK_JACOBI_CLUSTER"] = "1"
    run_v(rows, cols, False)
    del os.environ["EDAK_JACOBI_CLUSTER"]
