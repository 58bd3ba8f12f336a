"""cfg4: J trace of the benched pass (graph, 2 groups) vs a 1-group eager
solve, per iteration; exact J of both final x (edak_cost)."""
import numpy as np
import torch

import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_23571_b200 import build
build.build()
from paper_2605_23571_b200.engine import EdaPass
from paper_2605_23571_b200.krylov import pcg_members
from paper_2605_23571_b200.twin import BASELINE_CONFIGS, build_ensemble

dens = build_ensemble(BASELINE_CONFIGS[4])
eng = EdaPass(dens)
res = eng.run()
B = eng.rhs()
X1, t1 = pcg_members(eng.members, B[1:].contiguous(), eng.scfg, res.lmp, graph=False, groups=1)
J2 = np.array([t.cost for t in res.traces])
J1 = np.array([t.cost for t in t1])
R2 = np.array([t.resnorm for t in res.traces])
R1 = np.array([t.resnorm for t in t1])
d = np.abs(J1 - J2) / np.abs(J2)
print("max rel dJ per iteration:", np.array2string(d.max(0), precision=2))
m = int(np.unravel_index(d.argmax(), d.shape)[0])
print("worst member", m, "J2", J2[m, -5:], "J1", J1[m, -5:])
print("resnorm2", R2[m, ::8])
print("resnorm1", R1[m, ::8])
ex2 = eng.members.cost_members(res.x).cpu().numpy()
ex1 = eng.members.cost_members(X1).cpu().numpy()
print("exact J(x) vs identity, graph:", np.max(np.abs(ex2 - J2[:, -1]) / np.abs(ex2)))
print("exact J(x) vs identity, 1grp:", np.max(np.abs(ex1 - J1[:, -1]) / np.abs(ex1)))
print("exact J graph vs 1grp:", np.max(np.abs(ex1 - ex2) / np.abs(ex2)))
print("x rel diff", float((X1 - res.x).norm() / res.x.norm()))
print("lmp values", res.approx.values[:3], res.approx.values[-3:], "theta", res.lmp.theta)
