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

# hybrid storage (stream x1..x3, recompute x4) vs state-only recompute
if os.environ.get("HYBRID_AB", "1") == "1":
    from paper_2605_23571_b200.assim import Linearization
    from paper_2605_23571_b200.model import integrate_device
    for k in ("EDAK_SWEEP_V2", "EDAK_SWEEP_NOCHUNK", "EDAK_SWEEP_FAMILY"):
        os.environ.pop(k, None)
    st, sg = integrate_device(dens.x0, cfg.dt, cfg.n_steps, cfg.forcing, want_stages=True)
    hyb = Linearization(st, cfg.dt, cfg.forcing, dens.net, dens.ub, dens.rn, sg, "hybrid")
    rec = Linearization(st, cfg.dt, cfg.forcing, dens.net, dens.ub, dens.rn, None, "recompute")
    ct = torch.arange(1, ens.M + 1, dtype=torch.int32, device="cuda") % st.shape[0]
    for name, L in (("recompute", rec), ("hybrid", hyb)):
        o = L.tl_cols(V, ct)
        gg = L.ad_cols(W, ct)
        if name == "recompute":
            ro, rg = o, gg
        same = bool(torch.equal(o, ro)) and bool(torch.equal(gg, rg))
        t_tl = timeit(lambda: L.tl_cols(V, ct))
        t_ad = timeit(lambda: L.ad_cols(W, ct))
        t_h = timeit(lambda: L.hessian_cols(V, ct, 1.0))
        print(f"cfg{cfg.name[-1]} {name}: TL {t_tl:.3f} ms  AD {t_ad:.3f} ms  hessian {t_h:.3f} ms  "
              f"identical={same}", flush=True)
