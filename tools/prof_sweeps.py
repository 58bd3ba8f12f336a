"""Profiling driver: the cfg4 PCG-block sweeps (TL, AD, U_B) on 200 member
trajectories, a few launches each -- short enough for ncu --set full."""
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
eng = EdaPass(dens)
ens = eng.members
lin = ens.lin
V = torch.randn(ens.M, lin.n, dtype=torch.float64, device="cuda")
W = torch.randn(ens.M, lin.p, dtype=torch.float64, device="cuda")
for _ in range(3):
    lin.tl_cols(V, ens.traj_of)
    lin.ad_cols(W, ens.traj_of)
    lin.dfac.apply_cols(V)
    ens.a_apply_members(V, ident=1.0)
torch.cuda.synchronize()
print("ok")
