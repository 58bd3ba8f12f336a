"""U_B (overlap-save) on a config's member block, a few calls -- the program
an ncu capture of k_circ_os profiles (CFG env, default 4; MEMBERS cap)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2605_23571_b200 import build  # noqa: E402

build.build()
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

cfg = BASELINE_CONFIGS[int(os.environ.get("CFG", "4"))]
m = min(cfg.members, int(os.environ.get("MEMBERS", "100")))
dens = build_ensemble(cfg, members=2)
V = torch.randn(m, cfg.n, dtype=torch.float64, device="cuda")
for _ in range(4):
    dens.lin.dfac.apply_cols(V)
torch.cuda.synchronize()
print("done")
