"""TL/AD sweep time at cfg4 for stage_mode recompute vs hybrid (stored x1..x3
streamed, x4 recomputed), with a bit-identity check."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]


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


ref = None
for mode in ("recompute", "hybrid"):
    ens = EdaPass(build_ensemble(cfg, stage_mode=mode)).members
    lin = ens.lin
    g = torch.Generator(device="cuda").manual_seed(0)
    V = torch.randn(ens.M, lin.n, dtype=torch.float64, device="cuda", generator=g)
    W = torch.randn(ens.M, lin.p, dtype=torch.float64, device="cuda", generator=g)
    obs, gg = lin.tl_cols(V, ens.traj_of), lin.ad_cols(W, ens.traj_of)
    if ref is None:
        ref = (obs, gg)
    same = bool(torch.equal(obs, ref[0])) and bool(torch.equal(gg, ref[1]))
    t_tl = timeit(lambda: lin.tl_cols(V, ens.traj_of))
    t_ad = timeit(lambda: lin.ad_cols(W, ens.traj_of))
    print(f"{mode}: TL {t_tl:.3f} ms  AD {t_ad:.3f} ms  identical={same}", flush=True)
    del ens, lin
    torch.cuda.empty_cache()
