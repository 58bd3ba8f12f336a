"""One ensemble data-assimilation pass on the device -- the hot path of the
reference experiments (harness.py:178-182, 240-267) for a BASELINE config:

    b_j = rhs for control + every member        one batched AD launch
    Gamma = b_j - b_0 (+ Gaussian columns)      sketch.py:66-74
    Y = A_control Gamma, Nystrom EVD, LMP      nystrom.py:96-133, lmp.py:77-81
    PCG for every member with the control LMP  krylov.py:49-97 (batched)

``prepare`` builds the device state once; ``run`` executes a pass without
any host synchronisation until the traces are read back.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from .assim import Ensemble, TrajectoryOperator
from .krylov import SolverConfig, pcg_members
from .lmp import make_lmp
from .nystrom import NystromConfig, nystrom_evd
from .twin import substream


@dataclass
class PassResult:
    x: torch.Tensor        # (M, n) member increments z
    traces: list           # SolveTrace per member
    approx: object         # EigenApproximation of the control operator
    lmp: object
    gamma: torch.Tensor    # (ell, n) sketch


class EdaPass:
    """Device pipeline for one twin ensemble (control row 0 + members)."""

    def __init__(self, dens, pcg_iters=None, ell=None, k=None, theta_rule="halfsum",
                 trace_cost=True, cost="recurrence", member_offset=0, total_members=None,
                 distributed=False):
        self.dens = dens
        cfg = dens.cfg
        self.cfg = cfg
        self.ell = cfg.ell if ell is None else ell
        self.k = cfg.k if k is None else k
        self.iters = cfg.pcg_iters if pcg_iters is None else pcg_iters
        self.rule = theta_rule
        self.member_offset = member_offset
        self.total_members = dens.members if total_members is None else total_members
        self.distributed = distributed
        self.trace_cost = trace_cost
        self.cost = cost
        lin = dens.lin
        traj_of = np.asarray(dens.traj_of)
        self.all_rows = Ensemble(lin, dens.innovations, traj_of)
        self.control_row = Ensemble(lin, dens.innovations[:1], traj_of[:1])
        self.members = Ensemble(lin, dens.innovations[1:], traj_of[1:])
        self.control = TrajectoryOperator(lin, int(traj_of[0]))
        extra = self.ell - min(self.ell, self.total_members)
        self.gauss = None
        if extra > 0:  # cfg3: Gamma padded with Gaussian columns ("sketch" stream)
            g = substream(cfg.seed, "sketch").standard_normal((cfg.n, extra))
            self.gauss = _dev.f64(np.ascontiguousarray(g.T))
        self.ncfg = NystromConfig(ell=self.ell, k=self.k, shift_mode="trace")
        self.scfg = SolverConfig(max_iters=self.iters, trace_cost=trace_cost)

    def sketch(self, B):
        take = min(self.ell, self.total_members)
        if self.distributed:
            from .parallel import gather_sketch_rows
            G = gather_sketch_rows(B[1:] - B[0:1], self.member_offset, take)
        else:
            G = B[1: take + 1] - B[0:1]
        if self.gauss is not None:
            G = torch.cat([G, self.gauss], 0)
        return G.contiguous()

    def build_lmp(self, B):
        G = self.sketch(B)
        approx = nystrom_evd(self.control.a_apply, G.t(), self.ncfg)
        return G, approx, make_lmp(approx, self.rule)

    def rhs(self):
        """(M + 1, n) right-hand sides, row 0 the control's: the control and
        the member block are two launches into the same buffer, so a member's
        column position in every batched launch (the overlap-save U_B pairs
        columns 2c, 2c + 1 into one complex FFT) depends only on its member
        id, never on the control row -- the pass is then bit-identical under
        any even member sharding (tests/test_gpu_multirank.py)."""
        B = torch.empty((self.members.M + 1, self.cfg.n), dtype=torch.float64,
                        device=self.dens.innovations.device)
        self.control_row.rhs_all(out=B[:1])
        self.members.rhs_all(out=B[1:])
        return B

    def run(self, lmp=None):
        B = self.rhs()
        G, approx = None, None
        if lmp is None:
            G, approx, lmp = self.build_lmp(B)
        X, traces = pcg_members(self.members, B[1:].contiguous(), self.scfg, lmp, self.cost)
        return PassResult(X, traces, approx, lmp, G)

    @property
    def applies_per_pass(self):
        """Hessian-column applications per pass: ell sketch columns + one per
        member per PCG iteration (rhs sweeps are half-applies, not counted)."""
        return self.ell + self.dens.members * self.iters
