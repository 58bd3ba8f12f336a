"""Sketch matrices (mirrors reference ``sketch.py``).

``rhs_diff_sketch`` computes every member's right-hand side in ONE batched
adjoint launch (edak_rhs over all members, each with its own trajectory)
when the problems are our MemberProblems, and forms
Gamma_j = b_j - b_control on the device (sketch.py:66-74).  Every sketch
keeps its (ell, n) device block in ``device_columns`` so nystrom_evd does
not re-upload it.
"""

from dataclasses import dataclass

import numpy as np

from . import _dev

KINDS = ("gaussian", "power", "bcov", "bfactor", "rhsdiff")


@dataclass
class SketchMatrix:
    """sketch.py:30-40."""

    columns: np.ndarray
    kind: str
    n_build_matvecs: int = 0
    device_columns: object = None

    @property
    def ell(self):
        return self.columns.shape[1]


def gaussian_sketch(n, ell, rng):
    """sketch.py:43-45 (host RNG stream, as the reference)."""
    return SketchMatrix(rng.standard_normal((n, ell)), "gaussian", 0)


def power_sketch(prob, ell, rng):
    """sketch.py:48-51."""
    return SketchMatrix(prob.a_apply(rng.standard_normal((prob.n, ell))), "power", 1)


def bcov_sketch(ub, ell, rng):
    """sketch.py:54-57."""
    return SketchMatrix(ub.apply(ub.apply_t(rng.standard_normal((ub.n, ell)))), "bcov", 0)


def bfactor_sketch(ub, ell, rng):
    """sketch.py:60-63."""
    return SketchMatrix(ub.apply_t(rng.standard_normal((ub.n, ell))), "bfactor", 0)


def rhs_differences_device(ens, control_row=0):
    """Gamma block (M-1, n) on the device from an Ensemble whose member
    ``control_row`` is the control: one batched rhs launch."""
    B = ens.rhs_all()
    keep = [j for j in range(B.shape[0]) if j != control_row]
    return (B[keep] - B[control_row]).contiguous()


def rhs_diff_sketch(control, members):
    """Gamma_j = b_j - b_control (sketch.py:66-74)."""
    if hasattr(control, "lin") and all(hasattr(m, "lin") for m in members):
        from .assim import Ensemble
        ens = Ensemble.from_members([control, *members])
        G = rhs_differences_device(ens, 0)
        return SketchMatrix(G.t().cpu().numpy(), "rhsdiff", 0, device_columns=G)
    b0 = control.rhs()
    return SketchMatrix(np.column_stack([m.rhs() - b0 for m in members]), "rhsdiff", 0)


def make_sketch(kind, setup, ell, rng):
    """sketch.py:77-97."""
    if kind == "gaussian":
        return gaussian_sketch(setup.cfg.n, ell, rng)
    if kind == "power":
        return power_sketch(setup.control, ell, rng)
    if kind == "bcov":
        return bcov_sketch(setup.ub, ell, rng)
    if kind == "bfactor":
        return bfactor_sketch(setup.ub, ell, rng)
    if kind == "rhsdiff":
        if ell != len(setup.members):
            raise ValueError(
                f"rhsdiff sketch width is the ensemble size "
                f"({len(setup.members)}), got ell={ell}")
        return rhs_diff_sketch(setup.control, setup.members)
    raise ValueError(f"unknown sketch kind {kind!r}; expected one of {KINDS}")


def as_device(sketch):
    """(ell, n) device block of a SketchMatrix / ndarray."""
    dc = getattr(sketch, "device_columns", None)
    if dc is not None:
        return dc
    cols = np.asarray(getattr(sketch, "columns", sketch), dtype=float)
    return _dev.to_cols(cols, cols.shape[0])[0]
