"""A/B timing of the sweep kernel families on the cfg4 PCG block (or CFG)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
dens = build_ensemble(cfg)
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


ref_obs = ref_g = None
for fam in sys.argv[1:] or ["4,512", "4,256", "8,256", "8,128", "2,512"]:
    os.environ["EDAK_SWEEP_FAMILY"] = fam
    obs = lin.tl_cols(V, ens.traj_of)
    g = lin.ad_cols(W, ens.traj_of)
    if ref_obs is None:
        ref_obs, ref_g = obs, g
    same = bool(torch.equal(obs, ref_obs)) and bool(torch.equal(g, ref_g))
    t_tl = timeit(lambda: lin.tl_cols(V, ens.traj_of))
    t_ad = timeit(lambda: lin.ad_cols(W, ens.traj_of))
    print(f"family {fam}: TL {t_tl:.3f} ms  AD {t_ad:.3f} ms  identical={same}", flush=True)
