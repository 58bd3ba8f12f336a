"""A/B timing of sweep knobs on a config's PCG block (CFG env, default 4).

    python tools/ab_knobs.py "EDAK_SWEEP_DEPTH=1" "EDAK_TL_DEPTH=1+EDAK_AD_DEPTH=2" ...

Each argument is a "+"-separated set of environment assignments applied
before the launches (the library reads its knobs at launch time).  Prints TL,
AD and full Hessian-block times and whether the results are bit-identical to
the first variant's."""
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
gen = torch.Generator(device="cuda").manual_seed(0)
V = torch.randn(ens.M, lin.n, dtype=torch.float64, device="cuda", generator=gen)
W = torch.randn(ens.M, lin.p, dtype=torch.float64, device="cuda", generator=gen)


def timeit(fn, reps=20):
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
variants = sys.argv[1:] or [""]
keys = {kv.split("=")[0] for v in variants for kv in v.split("+") if kv}
for rnd in range(2):
    for v in variants:
        for k in keys:
            os.environ.pop(k, None)
        for kv in v.split("+"):
            if kv:
                k, val = kv.split("=")
                os.environ[k] = val
        obs = lin.tl_cols(V, ens.traj_of)
        g = lin.ad_cols(W, ens.traj_of)
        h = ens.a_apply_members(V, ident=1.0)
        if ref is None:
            ref = (obs, g, h)
        same = all(bool(torch.equal(a, b)) for a, b in zip((obs, g, h), ref))
        t_tl = timeit(lambda: lin.tl_cols(V, ens.traj_of))
        t_ad = timeit(lambda: lin.ad_cols(W, ens.traj_of))
        t_h = timeit(lambda: ens.a_apply_members(V, ident=1.0))
        t_u = timeit(lambda: lin.dfac.apply_cols(V))
        print(f"cfg{cfg.name[-1]} [{v or 'default'}] round {rnd}: TL {t_tl:.4f} ms  AD {t_ad:.4f} ms  "
              f"U_B {t_u:.4f} ms  hessian {t_h:.4f} ms  identical={same}", flush=True)
