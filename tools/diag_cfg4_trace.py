"""cfg4 member trace diagnostics: identity J vs exact J of the iterate (GPU
edak_cost) vs the oracle trace, per iteration, for members in both groups."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
from paper_2605_23571_b200 import build  # noqa: E402
build.build()
from oracle import algorithms as oalg  # noqa: E402
from parity import oracle_rows  # noqa: E402
from paper_2605_23571_b200.assim import Ensemble  # noqa: E402
from paper_2605_23571_b200.engine import EdaPass  # noqa: E402
from paper_2605_23571_b200.krylov import SolverConfig, pcg_members  # noqa: E402
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble  # noqa: E402

dens = build_ensemble(BASELINE_CONFIGS[4])
eng = EdaPass(dens)
res = eng.run()
B = eng.rhs()
rows = [1, 100, 101, 200]
sub = Ensemble(dens.lin, dens.innovations[rows], np.asarray(dens.traj_of)[rows])
snaps = []
X, trs = pcg_members(sub, B[rows].contiguous(), SolverConfig(max_iters=80), res.lmp, snapshots=snaps)
Jex = np.array([sub.cost_members(s[1]).cpu().numpy() for s in snaps]).T  # (4, 81)
ops = oracle_rows(dens, rows)
olmp = oalg.SpectralLmp(res.approx.vectors, res.approx.values, res.lmp.theta)
np.set_printoptions(linewidth=200, precision=6)
for i, (r, op) in enumerate(zip(rows, ops)):
    xr, ref = oalg.pcg(op.hessian_apply, op.rhs(), oalg.SolverConfig(max_iters=80), precond=olmp,
                       cost_fn=op.quadratic_cost)
    Jb = np.array(res.traces[r - 1].cost)
    Jid = np.array(trs[i].cost)
    Jr = np.array(ref.cost)
    print(f"row {r}: bench-vs-ref rel", np.abs(Jb - Jr)[:40] / Jr[:40])
    print(f"row {r}: snapG1 identity-vs-exact rel", np.abs(Jid - Jex[i])[:40] / Jex[i][:40])
    print(f"row {r}: snapG1 exact-vs-ref rel", np.abs(Jex[i] - Jr)[:40] / Jr[:40])
    print(f"row {r}: resnorm ours", np.array(trs[i].resnorm)[15:30])
    print(f"row {r}: resnorm ref ", np.array(ref.resnorm)[15:30])
    print(f"row {r}: J ref", Jr[15:30])
