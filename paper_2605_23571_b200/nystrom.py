"""Randomized Nystrom EVD on the GPU (mirrors reference ``nystrom.py``).

Same API, dataclasses, validation and exceptions as the reference
(nystrom.py:31-145).  The algorithm is the reference's pass
    Y = A Phi;  W = Phi^T Y;  W = C^T C (shifted on breakdown);
    A_N = F F^T with F = Y C^-1;  S, D = leading left singular pairs of F
(the reference reaches the same F through Q_Y (R_Y C^-1), nystrom.py:118-131)
with every dense step on the device:

* W = Phi^T Y, Gram matrices: DMMA split-K GEMM (edak_gemm_tn);
* Cholesky with the identical nu schedule and dpotrf breakdown test
  (edak_potrf_shifted), C^-1 (edak_trinv_upper);
* tall, large n: CholeskyQR2 of Y (DMMA Grams and triangular solves as
  GEMMs; a third pass only when the second Cholesky factor is not close to
  I, the shifted CholeskyQR3 when a Gram is not numerically SPD), T =
  R_Y C^-1, one-sided Jacobi SVD of the l x l T, S = Q_Y U_T with the last
  pass's triangular solve applied to U_T instead of to the n x l basis;
* small n, wide (l > n, cfg2) or when CholeskyQR2's Gram is not positive
  definite: one-sided Jacobi SVD straight on F (or F^T when l > n),
  which handles exact rank deficiency.
The rank check (nystrom.py:136-140) raises for exactly-zero columns of Y,
the case in which Householder's R_Y has an exactly zero diagonal.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from .linalg import chol_blocked, chol_inv, col_dots, gemm_nn, gemm_tn, svd_jacobi

SHIFT_MODES = (None, "trace", "ynorm")
_MODE_CODE = {None: 0, "trace": 1, "ynorm": 2}
QR_MIN_ASPECT = 4
QR_MIN_N = 256


class NystromBreakdownError(RuntimeError):
    """Sketch does not support a usable factorization (nystrom.py:31)."""


@dataclass
class NystromConfig:
    """nystrom.py:35-50."""

    ell: int
    k: int
    q: int = 1
    shift_mode: str | None = None

    def __post_init__(self):
        if not 1 <= self.k <= self.ell:
            raise ValueError(f"need 1 <= k <= ell, got k={self.k} ell={self.ell}")
        if self.q < 1:
            raise ValueError(f"need q >= 1, got {self.q}")
        if self.shift_mode not in SHIFT_MODES:
            raise ValueError(f"shift_mode must be one of {SHIFT_MODES}")


class EigenApproximation:
    """nystrom.py:53-64.  ``device_vectors`` keeps the (k, n) device block;
    the numpy ``vectors`` (n, k) are downloaded on first access only."""

    def __init__(self, vectors=None, values=None, shift=0.0, n_build_matvecs=0,
                 device_vectors=None):
        self._vectors = None if vectors is None else np.asarray(vectors, dtype=float)
        self.values = np.asarray(values, dtype=float)
        self.shift = shift
        self.n_build_matvecs = n_build_matvecs
        self.device_vectors = device_vectors

    @property
    def vectors(self):
        if self._vectors is None and self.device_vectors is not None:
            self._vectors = self.device_vectors.t().cpu().numpy()
        return self._vectors

    @vectors.setter
    def vectors(self, v):
        self._vectors = np.asarray(v, dtype=float)

    @property
    def k(self):
        return self.values.size

    def __repr__(self):
        return (f"EigenApproximation(k={self.k}, values={self.values!r}, "
                f"shift={self.shift!r}, n_build_matvecs={self.n_build_matvecs})")


def shifted_cholesky(w, mode, scale):
    """Upper Cholesky factor of ``w``, shifted on breakdown if allowed
    (nystrom.py:67-93): the plain factorization first, then w + nu I with
    nu = eps * scale grown by factors of 10 (5 tries) when ``mode`` is not
    None.  Returns ``(c, nu_used)``; raises NystromBreakdownError with the
    reference's messages.  On the device (edak_potrf_shifted, dpotrf's
    breakdown test); numpy in, numpy out."""
    from .linalg import potrf_shifted
    w = np.asarray(w, dtype=float)
    if w.ndim != 2 or w.shape[0] != w.shape[1]:
        raise ValueError("shifted_cholesky needs a square matrix")
    # the block layout holds columns contiguously: the transpose of numpy's rows
    W = _dev.f64(np.ascontiguousarray(w.T))
    code = 0 if mode is None else 2  # 2: nu0 = eps * scale with the caller's scale
    Cm, nu, info = potrf_shifted(W, code, float(scale))
    info = info.cpu().numpy()
    if info[1]:
        if info[0] <= 1:
            raise NystromBreakdownError(
                "Cholesky of the sketched Gram matrix broke down and no "
                "usable shift is available")
        raise NystromBreakdownError("sketched Gram matrix stayed indefinite after shifting")
    return Cm.cpu().numpy().T.copy(), float(nu[0])


def _device_owner(a_apply):
    """Our operator object when a_apply is its bound ``a_apply`` (then the
    sketch never leaves the device)."""
    owner = getattr(a_apply, "__self__", None)
    if hasattr(owner, "a_apply_cols") and getattr(a_apply, "__name__", "") == "a_apply":
        return owner
    return None


def _apply_block(a_apply, phi_cols, n):
    owner = _device_owner(a_apply)
    if owner is not None:
        return owner.a_apply_cols(phi_cols)
    y = a_apply(phi_cols.t().cpu().numpy())
    cols, _, _ = _dev.to_cols(np.asarray(y, dtype=float).reshape(n, -1), n)
    return cols


def _check_rank(Y):
    nrm = col_dots(Y, Y).cpu().numpy()
    dead = np.flatnonzero(nrm == 0.0)
    if dead.size:
        raise NystromBreakdownError(f"sketch column {dead[0]} was annihilated by the operator")


def _cholqr_pass(Y, shift=0.0):
    """One CholeskyQR pass: R = chol(Y^T Y + shift I), Q = Y R^-1 (DMMA
    Grams / products); info[1] != 0 when the Gram was not numerically SPD."""
    G = gemm_tn(Y, Y)
    if shift:
        G.diagonal().add_(shift)
    R, Rinv, _, info = chol_inv(G, 0)
    return gemm_nn(Y, Rinv), R, info


def _cholqr2(Y):
    """Q (l, n) block and upper R (l, l) block with Y = Q R by shifted
    CholeskyQR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa, SIAM J.
    Sci. Comput. 2020): a first pass on Y^T Y + s I, s = 11 (m l + l (l+1))
    u ||Y||_F^2 -- SPD for any cond(Y) < u^-1 -- then CholeskyQR2 of its Q.
    Orthogonality and residual end at the u level, like the reference's
    Householder QR (nystrom.py:118); every pass is two DMMA GEMMs plus an
    (l x l) Cholesky / triangular inverse.  None only if a Gram broke down."""
    l, m = Y.shape
    tr = float(col_dots(Y, Y).sum())
    s = 11.0 * (m * l + l * (l + 1)) * np.finfo(float).eps * tr
    Q, R, info = _cholqr_pass(Y, s)
    if int(info[1]):
        return None
    for _ in range(2):
        Q, R2, info = _cholqr_pass(Q)
        if int(info[1]):
            return None
        R = gemm_nn(R2, R)  # upper R_k ... R_1
    return Q, R


ORTHO_TOL = 0.1   # ||R_k - I||_F below which the pass's input basis counts as orthonormal
MAX_PLAIN = 4     # unshifted CholeskyQR passes before the shifted CholeskyQR3 takes over


def _cholqr_lazy(Y, extra=()):
    """Y = Q_Y R_Y with Q_Y = Qp Ti and R_Y = R, for blocks Qp (l, n),
    the last pass's triangular inverse Ti (l, l) and R (l, l) upper, so the
    caller forms Q_Y U only as Qp (Ti U) and never materialises Q_Y (the
    n x l x l product of the last pass).

    Unshifted CholeskyQR passes Q_k = Q_{k-1} R_k^-1 until the Cholesky
    factor R_k of a pass's Gram is within ORTHO_TOL of I in Frobenius norm:
    then its input Q_{k-1} has cond <= (1 + tol) / (1 - tol) and CholeskyQR
    of it is orthonormal to O(u cond^2) = O(u) (Yamamoto, Nakatsukasa,
    Yanagisawa, Fukaya, ETNA 2015), the level of the reference's
    Householder QR (nystrom.py:118).  A well-conditioned sketch takes two
    passes (CholeskyQR2) instead of shifted CholeskyQR3's three; a Gram that
    is not numerically SPD (cond(Y) >~ u^-1/2), or no convergence in
    MAX_PLAIN passes, falls back to the shifted CholeskyQR3 (_cholqr2).

    The first two passes run without a host read; ONE read then fetches
    their breakdown flags, the deviation of R_2 and the ``extra`` device
    tensors (returned as a host array).  Returns (qr or None, extra)."""
    l = Y.shape[0]
    eye = torch.eye(l, dtype=Y.dtype, device=Y.device)
    R1, R1i, _, i1 = chol_inv(gemm_tn(Y, Y), 0, defer=True)
    Q1 = gemm_nn(Y, R1i)
    R2, R2i, _, i2 = chol_inv(gemm_tn(Q1, Q1), 0, defer=True)
    dev = torch.linalg.matrix_norm(R2 - eye)
    chk = torch.cat([i1.to(torch.float64), i2.to(torch.float64), dev.view(1)]
                    + [e.to(torch.float64).reshape(-1) for e in extra]).cpu().numpy()
    host = chk[5:]
    ok = not chk[1] and not chk[3] and np.isfinite(chk[4])
    if ok:
        R = gemm_nn(R2, R1)  # upper R_2 R_1
        if chk[4] <= ORTHO_TOL:
            return (Q1, R2i, R), host
        Q = gemm_nn(Q1, R2i)
        for _ in range(MAX_PLAIN - 2):
            Rk, Rki, _, info = chol_inv(gemm_tn(Q, Q), 0)
            dk = torch.linalg.matrix_norm(Rk - eye)
            c = torch.cat([info.to(torch.float64), dk.view(1)]).cpu().numpy()
            if c[1] or not np.isfinite(c[2]):
                break
            R = gemm_nn(Rk, R)
            if c[2] <= ORTHO_TOL:
                return (Q, Rki, R), host
            Q = gemm_nn(Q, Rki)
    qr = _cholqr2(Y)
    if qr is None:
        return None, host
    return (qr[0], eye, qr[1]), host


_SIDE = {}


def _side_stream():
    dev = torch.cuda.current_device()
    if dev not in _SIDE:
        _SIDE[dev] = torch.cuda.Stream()
    return _SIDE[dev]


def _use_qr(n, ell):
    """Tall sketches go through CholeskyQR + an (l x l) Jacobi SVD; short or
    wide ones (n < 4 l, e.g. cfg2's l = 50 > n = 40) through a Jacobi SVD
    of the whole F, which also covers exact rank deficiency."""
    return n >= QR_MIN_ASPECT * ell and n >= QR_MIN_N


def _orthobasis(Y):
    """Orthonormal basis of range(Y) for the q > 1 passes."""
    n = Y.shape[1]
    if _use_qr(n, Y.shape[0]):
        qr = _cholqr2(Y)
        if qr is not None:
            return qr[0]
    if n >= Y.shape[0]:
        return svd_jacobi(Y)[0]
    U, _, V = svd_jacobi(Y.t().contiguous(), want_v=True)
    return V


def nystrom_evd(a_apply, sketch, cfg):
    """Leading eigenpairs of an SPD operator (nystrom.py:96-133)."""
    phi_in = getattr(sketch, "columns", sketch)
    dev_phi = getattr(sketch, "device_columns", None)
    if isinstance(phi_in, torch.Tensor):
        n, ell = phi_in.shape
        phi = phi_in.to(_dev.device(), torch.float64).t().contiguous()
    else:
        phi_np = np.asarray(phi_in, dtype=float)
        n, ell = phi_np.shape
        phi = dev_phi if dev_phi is not None else _dev.to_cols(phi_np, n)[0]
    if ell != cfg.ell:
        raise ValueError(f"sketch has {ell} columns, cfg.ell={cfg.ell}")
    Y = _apply_block(a_apply, phi, n)
    if cfg.q > 1:
        _check_rank(Y)
    for _ in range(cfg.q - 1):
        phi = _orthobasis(Y)
        Y = _apply_block(a_apply, phi, n)
        _check_rank(Y)
    mode = _MODE_CODE[cfg.shift_mode]
    scale = 0.0
    if cfg.shift_mode == "ynorm":
        scale = float(torch.sqrt(col_dots(Y, Y).sum()))
    k_eff = min(cfg.k, ell, n)
    ydots = col_dots(Y, Y)  # the rank check (nystrom.py:136-140), read with the QR flags
    use_qr = _use_qr(n, ell)
    # W = Phi^T Y and its shifted Cholesky (nystrom.py:125-127) on a side
    # stream, overlapping the CholeskyQR passes of Y on the main stream
    main = torch.cuda.current_stream()
    side = _side_stream() if use_qr else main
    ready = torch.cuda.Event()
    ready.record(main)
    with torch.cuda.stream(side):
        side.wait_event(ready)
        W = gemm_tn(phi, Y)  # block (l, l): W[a][b] = phi_a . y_b
        Cm, Cinv, nu, winfo = chol_inv(W, mode, scale, defer=True)
        wdone = torch.cuda.Event()
        wdone.record(side)
    main.wait_event(wdone)
    if use_qr:
        qr, host = _cholqr_lazy(Y, extra=(ydots, winfo, nu))
    else:
        qr, host = None, torch.cat([ydots, winfo.to(torch.float64), nu]).cpu().numpy()
    dead = np.flatnonzero(host[:ell] == 0.0)
    if dead.size:
        raise NystromBreakdownError(f"sketch column {dead[0]} was annihilated by the operator")
    info, shift = host[ell:ell + 2], float(host[ell + 2])
    if info[1] and chol_blocked(ell) and mode != 0:
        # the deferred 2 x 2 block factorisation broke down: the one-kernel
        # factorisation with the reference's shift schedule from the start
        Cm, Cinv, nu, winfo = chol_inv(W, mode, scale, single=True)
        info, shift = winfo.cpu().numpy(), float(nu[0])
    if info[1]:
        if info[0] <= 1:
            raise NystromBreakdownError(
                "Cholesky of the sketched Gram matrix broke down and no "
                "usable shift is available")
        raise NystromBreakdownError("sketched Gram matrix stayed indefinite after shifting")
    if qr is not None:
        Qp, Ti, R = qr
        T = gemm_nn(R, Cinv)                 # R_Y C^-1 (l x l)
        U_T, sig, _ = svd_jacobi(T)
        S = gemm_nn(Qp, gemm_nn(Ti, U_T[:k_eff].contiguous()))  # Q_Y U_T[:, :k] = Qp (Ti U_T[:, :k])
    else:
        F = gemm_nn(Y, Cinv)                 # Y C^-1 (n x l)
        if n >= ell:
            U, sig, _ = svd_jacobi(F)
            S = U[:k_eff]
        else:
            _, sig, V = svd_jacobi(F.t().contiguous(), want_v=True)
            S = V[:k_eff]
    S = S.contiguous()
    values = (sig[:k_eff] ** 2).cpu().numpy()
    return EigenApproximation(values=values, shift=shift, n_build_matvecs=cfg.q,
                              device_vectors=S)


def reconstruct(approx):
    """S diag(D) S^T (nystrom.py:143-145)."""
    return (approx.vectors * approx.values) @ approx.vectors.T
