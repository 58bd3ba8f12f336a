"""Persistent small-n PCG vs the batched path and the oracle: J / resnorm
distance per iteration, and the paths' own sensitivity to 1e-16 input jitter."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from oracle import algorithms as oalg
from oracle.twin import TwinConfig, build_setup
from paper_2605_23571_b200.assim import Ensemble, MemberProblem
from paper_2605_23571_b200.krylov import SolverConfig, pcg_members

tw = TwinConfig(n=40, obs_grid_count=8, members=7)
setup = build_setup(tw, trial_seed=1)
mems = [MemberProblem(m.traj, m.net, m.ub, m.rn, m.innovation) for m in setup.members]
ens = Ensemble.from_members(mems)
B = ens.rhs_all()
cfg = SolverConfig(max_iters=15)
om = setup.members[0]
_, ref = oalg.pcg(om.hessian_apply, om.rhs(), cfg, cost_fn=om.quadratic_cost)
Jr = np.array(ref.cost)
rr = np.array(ref.resnorm)
np.set_printoptions(precision=2, linewidth=200)
for small in (False, True):
    _, t = pcg_members(ens, B, cfg, small=small, graph=False)
    print("small" if small else "batch", "dJ", np.abs(np.array(t[0].cost) - Jr) / Jr)
    print("      dr", np.abs(np.array(t[0].resnorm) - rr) / rr[0])
    g = torch.Generator(device="cuda").manual_seed(0)
    for trial in range(3):
        Bp = B * (1 + 1e-16 * torch.randn(B.shape, generator=g, device="cuda", dtype=torch.float64))
        _, tp = pcg_members(ens, Bp, cfg, small=small, graph=False)
        print("   jit dJ", np.abs(np.array(tp[0].cost) - np.array(t[0].cost)) / Jr)
