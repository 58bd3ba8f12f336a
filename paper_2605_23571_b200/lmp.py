"""Scaled spectral LMP on the GPU (mirrors reference ``lmp.py``).

P = I + S (theta (Lambda + I)^-1 - I) S^T with symmetric factor
U = I + S (sqrt(theta) (Lambda + I)^-1/2 - I) S^T (lmp.py:1-16).
Each factor application is two DMMA GEMMs (edak_lmp_apply: W = S^T R,
Z = R + S diag(c) W) over a whole (ncols, n) block of member residuals.

``apply`` keeps the reference's two-factor form P v = U (U v)
(lmp.py:72-74) unless S is orthonormal to 1e-13 (checked once on the
device), in which case it applies P in one pass with c = theta/(lam+1) - 1
-- the fused "I + U diag(.) U^T" of the north star, equal to the two-pass
form up to rounding.
"""

import numpy as np
import torch

from . import _dev, _lib
from .linalg import gemm_tn

THETA_RULES = ("halfsum", "lambdak", "one")
ORTHO_TOL = 1e-13


def choose_theta(rule, lam_k_of_system):
    """lmp.py:25-41."""
    if lam_k_of_system < 1.0 - 1e-8:
        raise ValueError(f"I + A has eigenvalues >= 1, got lam_k={lam_k_of_system}")
    if rule == "halfsum":
        return 0.5 * (lam_k_of_system + 1.0)
    if rule == "lambdak":
        return float(lam_k_of_system)
    if rule == "one":
        return 1.0
    raise ValueError(f"unknown theta rule {rule!r}; expected {THETA_RULES}")


class SpectralLmp:
    """Preconditioner data (lmp.py:44-74) with device-resident S.

    ``vectors`` (n, k) numpy as in the reference, or None when
    ``device_vectors`` (k, n) is given (downloaded lazily)."""

    def __init__(self, vectors, values, theta, device_vectors=None, fused=None):
        if theta <= 0:
            raise ValueError("theta must be positive")
        self.values = np.asarray(values, dtype=float)
        if np.any(self.values < -1e-12):
            raise ValueError("eigenvalue estimates of A must be >= 0")
        self.theta = theta
        self._vectors = None if vectors is None else np.asarray(vectors, dtype=float)
        self.device_vectors = device_vectors
        self.fused = fused
        self._ready = False
        self.n = (self._vectors.shape[0] if self._vectors is not None
                  else int(device_vectors.shape[1]))

    @property
    def vectors(self):
        if self._vectors is None:
            self._vectors = self.device_vectors.t().cpu().numpy()
        return self._vectors

    @property
    def k(self):
        return self.values.size

    def _prepare(self):
        if self._ready:
            return
        S = self.device_vectors
        if S is None:
            S = _dev.to_cols(self._vectors, self.n)[0]
        self._S = S.contiguous()
        lam = np.asarray(self.values, dtype=float)
        self._c_sqrt = _dev.f64(np.sqrt(self.theta / (lam + 1.0)) - 1.0)
        self._c_full = _dev.f64(self.theta / (lam + 1.0) - 1.0)
        if self.fused is None:
            g = gemm_tn(self._S, self._S)
            eye = torch.eye(self.k, dtype=torch.float64, device=g.device)
            self.fused = bool((g - eye).abs().max() <= ORTHO_TOL)
        self._ready = True

    def single_pass(self):
        """(S (k, n), c = theta/(lam+1) - 1) when P is applied in one pass
        (S orthonormal), else None.  Batched PCG then folds P into its beta
        step (edak_pcg_lmp_beta) instead of materialising z = P r."""
        self._prepare()
        return (self._S, self._c_full) if self.fused else None

    def work_cols(self, ncols, device):
        """Split-K workspace of edak_lmp_apply, one per (ncols, device, stream):
        member groups of the batched PCG apply P on their own streams at the
        same time, so a workspace shared across streams would race."""
        key = (ncols, str(device), torch.cuda.current_stream(device).cuda_stream)
        cache = self.__dict__.setdefault("_work", {})
        w = cache.get(key)
        if w is None:
            w = torch.empty(int(_lib.lib().edak_lmp_work_doubles(self.n, self.k, ncols)),
                            dtype=torch.float64, device=device)
            cache[key] = w
        return w

    def _project_cols(self, coef, R, out=None):
        n, ncols = R.shape[1], R.shape[0]
        R = R.contiguous()
        out = torch.empty_like(R) if out is None else out
        work = self.work_cols(ncols, R.device)
        _lib.call("edak_lmp_apply", n, self.k, ncols, self._S.data_ptr(), coef.data_ptr(),
                  R.data_ptr(), out.data_ptr(), work.data_ptr(), _lib.stream())
        return out

    def apply_sqrt_cols(self, R, out=None):
        """U R for a (ncols, n) device block (lmp.py:67-70)."""
        self._prepare()
        return self._project_cols(self._c_sqrt, R, out)

    def apply_cols(self, R, out=None):
        """P R for a (ncols, n) device block (lmp.py:72-74)."""
        self._prepare()
        if self.fused:
            return self._project_cols(self._c_full, R, out)
        return self._project_cols(self._c_sqrt, self._project_cols(self._c_sqrt, R), out)

    def apply_sqrt(self, v):
        cols, vec, as_np = _dev.to_cols(v, self.n)
        return _dev.from_cols(self.apply_sqrt_cols(cols), vec, as_np)

    def apply(self, v):
        cols, vec, as_np = _dev.to_cols(v, self.n)
        return _dev.from_cols(self.apply_cols(cols), vec, as_np)


def make_lmp(approx, rule):
    """lmp.py:77-81."""
    theta = choose_theta(rule, float(approx.values[-1]) + 1.0)
    dv = getattr(approx, "device_vectors", None)
    return SpectralLmp(None if dv is not None else approx.vectors, approx.values, theta,
                       device_vectors=dv)
