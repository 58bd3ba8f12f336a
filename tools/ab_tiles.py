"""A/B of sweep tile family / window chunk (env knobs) on the cfg4 PCG block."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
ens = EdaPass(build_ensemble(cfg)).members
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


ref = None
for mode in sys.argv[1:]:
    for k in ("EDAK_SWEEP_FAMILY", "EDAK_SWEEP_CHUNK"):
        os.environ.pop(k, None)
    fam, chunk = mode.split("/")
    if fam != "default":
        os.environ["EDAK_SWEEP_FAMILY"] = fam
    os.environ["EDAK_SWEEP_CHUNK"] = chunk
    obs = lin.tl_cols(V, ens.traj_of)
    g = lin.ad_cols(W, ens.traj_of)
    if ref is None:
        ref = (obs, g)
    same = bool(torch.equal(obs, ref[0])) and bool(torch.equal(g, ref[1]))
    t_tl = timeit(lambda: lin.tl_cols(V, ens.traj_of))
    t_ad = timeit(lambda: lin.ad_cols(W, ens.traj_of))
    print(f"{mode}: TL {t_tl:.3f} ms  AD {t_ad:.3f} ms  sum {t_tl + t_ad:.3f}  identical={same}",
          flush=True)
