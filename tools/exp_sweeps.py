"""Sweep timing with experimental (wrong-by-design) library builds, to bound
what barriers / global loads cost: python tools/exp_sweeps.py <lib.so>..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import _lib, build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

dens = build_ensemble(BASELINE_CONFIGS[4])
ens = EdaPass(dens).members
lin = ens.lin
V = torch.randn(ens.M, lin.n, dtype=torch.float64, device="cuda")
W = torch.randn(ens.M, lin.p, dtype=torch.float64, device="cuda")


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for path in ["default"] + sys.argv[1:]:
    if path != "default":
        _lib._LIB = _lib.load(path)
    t_tl = timeit(lambda: lin.tl_cols(V, ens.traj_of))
    t_ad = timeit(lambda: lin.ad_cols(W, ens.traj_of))
    print(f"{path}: TL {t_tl:.3f} ms  AD {t_ad:.3f} ms", flush=True)
