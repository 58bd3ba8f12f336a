"""A/B timing of sweep implementations on a config's PCG block (CFG env,
default 4): first-generation register kernels (EDAK_SWEEP_V1) vs the
shared-memory-staged k_tl2/k_ad2, with bit-identity checks."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
dens = build_ensemble(cfg, members=min(cfg.members, int(os.environ.get("MEMBERS", "100000"))))
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


ref = None
modes = sys.argv[1:] or ["v1", "v2"]
for mode in modes:
    for k in ("EDAK_SWEEP_V2", "EDAK_SWEEP_NOCHUNK", "EDAK_SWEEP_FAMILY", "EDAK_TL_MINB",
              "EDAK_AD_MINB"):
        os.environ.pop(k, None)
    for part in mode.split("+")[1:]:          # e.g. v1+tl4+ad3
        if part.startswith("tl"):
            os.environ["EDAK_TL_MINB"] = part[2:]
        if part.startswith("ad"):
            os.environ["EDAK_AD_MINB"] = part[2:]
    if mode.startswith("v2"):
        os.environ["EDAK_SWEEP_V2"] = "1"
    if "nochunk" in mode:
        os.environ["EDAK_SWEEP_NOCHUNK"] = "1"
    obs = lin.tl_cols(V, ens.traj_of)
    g = lin.ad_cols(W, ens.traj_of)
    if ref is None:
        ref = (obs, g)
    same = bool(torch.equal(obs, ref[0])) and bool(torch.equal(g, ref[1]))
    t_tl = timeit(lambda: lin.tl_cols(V, ens.traj_of))
    t_ad = timeit(lambda: lin.ad_cols(W, ens.traj_of))
    t_h = timeit(lambda: ens.a_apply_members(V, ident=1.0))
    print(f"cfg{cfg.name[-1]} {mode}: TL {t_tl:.3f} ms  AD {t_ad:.3f} ms  hessian {t_h:.3f} ms  "
          f"identical={same}", flush=True)
