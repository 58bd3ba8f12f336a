"""Thin host wrappers over the dense fp64 entry points of libedak.so
(DMMA GEMMs, Cholesky with the reference shift schedule, triangular
inverse, one-sided Jacobi SVD, column dots).  Blocks are (ncols, rows)
device tensors = column-major (rows x ncols) matrices."""

import torch

from . import _lib


def _empty(*shape, like):
    return torch.empty(shape, dtype=torch.float64, device=like.device)


def gemm_tn(A, B):
    """A^T B for column blocks A (m, K), B (nb, K) -> (nb, m) block, i.e. the
    column-major (m x nb) matrix C[a, b] = A[a] . B[b]."""
    A, B = A.contiguous(), B.contiguous()
    m, K = A.shape
    nb = B.shape[0]
    C = _empty(nb, m, like=A)
    part = _empty(int(_lib.lib().edak_gemm_tn_partials(m, nb, K)), like=A)
    _lib.call("edak_gemm_tn", A.data_ptr(), K, B.data_ptr(), K, C.data_ptr(), m, m, nb, K,
              part.data_ptr(), _lib.stream())
    return C


def gemm_nn(A, B, bscale=None, Cin=None, beta=1.0, out=None):
    """out = beta * Cin + A diag(bscale) B with A a column block (kk, M)
    (column-major M x kk) and B a column block (N, kk): result (N, M)."""
    A, B = A.contiguous(), B.contiguous()
    kk, M = A.shape
    N = B.shape[0]
    out = _empty(N, M, like=A) if out is None else out
    _lib.call("edak_gemm_nn", A.data_ptr(), M, B.data_ptr(), kk, _lib.ptr(bscale),
              _lib.ptr(Cin), M, float(beta), out.data_ptr(), M, M, N, kk, _lib.stream())
    return out


def col_dots(A, B):
    A, B = A.contiguous(), B.contiguous()
    out = _empty(A.shape[0], like=A)
    _lib.call("edak_col_dots", A.shape[1], A.shape[0], A.data_ptr(), B.data_ptr(),
              out.data_ptr(), _lib.stream())
    return out


def potrf_shifted(W, mode, scale=0.0):
    """Upper Cholesky of the (l x l) column-major W (block (l, l)) with the
    nystrom.py:67-93 schedule.  Returns (C block, nu tensor[1], info int32[2])
    -- no host sync."""
    W = W.contiguous()
    l = W.shape[0]
    Cm = torch.zeros_like(W)
    nu = _empty(1, like=W)
    info = torch.zeros(2, dtype=torch.int32, device=W.device)
    _lib.call("edak_potrf_shifted", W.data_ptr(), l, Cm.data_ptr(), int(mode), float(scale),
              nu.data_ptr(), info.data_ptr(), _lib.stream())
    return Cm, nu, info


BLOCK_L = 128  # the register-resident Cholesky-inverse kernel's limit


def _chol_inv_2x2(W, defer=False):
    """Unshifted upper Cholesky W = C^T C and C^-1 of a 129..256 Gram as a
    2 x 2 block factorisation over the register kernel (l <= 128) and DMMA
    GEMMs (dpotrf's blocked right-looking order):
        C11 = chol(W11), C12 = C11^-T W12, C22 = chol(W22 - C12^T C12),
        C^-1 = [[C11^-1, -C11^-1 C12 C22^-1], [0, C22^-1]].
    Returns (C, C^-1, nu = 0, info) or None when a pivot broke down (the
    caller then runs the single-kernel factorisation with its shift
    schedule from the start, nystrom.py:67-93).  One host read of the two
    breakdown flags -- or, with ``defer``, none: the factors are returned
    whatever happened and info[1] != 0 flags a breakdown on the device."""
    l, h = W.shape[0], BLOCK_L
    m = l - h
    W11, W12, W22 = W[:h, :h].contiguous(), W[h:, :h].contiguous(), W[h:, h:].contiguous()
    C11, C11i, _, info1 = chol_inv(W11, 0)
    C12 = gemm_tn(C11i, W12)                      # C11^-T W12 (h x m): block (m, h)
    S = W22 - gemm_tn(C12, C12)                   # W22 - C12^T C12
    C22, C22i, _, info2 = chol_inv(S.contiguous(), 0)
    if not defer and (int(info1[1]) or int(info2[1])):
        return None
    X = gemm_nn(C11i, gemm_nn(C12, C22i))          # C11^-1 C12 C22^-1 (h x m): block (m, h)
    C = torch.zeros_like(W)
    Ci = torch.zeros_like(W)
    C[:h, :h], C[h:, :h], C[h:, h:] = C11, C12, C22
    Ci[:h, :h], Ci[h:, :h], Ci[h:, h:] = C11i, -X, C22i
    nu = torch.zeros(1, dtype=torch.float64, device=W.device)
    info = torch.maximum(info1, info2) if defer else torch.zeros(2, dtype=torch.int32, device=W.device)
    return C, Ci, nu, info


def chol_blocked(l):
    """True when chol_inv factors an l x l Gram by the 2 x 2 block path."""
    import os
    return BLOCK_L < l <= 2 * BLOCK_L and os.environ.get("EDAK_CHOL_BLOCKED", "1") != "0"


def chol_inv(W, mode, scale=0.0, want_inv=True, defer=False, single=False):
    """Fused blocked Cholesky + inverse (edak_chol_inv): (C, C^-1 or None,
    nu tensor[1], info int32[2]) with potrf_shifted's schedule -- no host
    sync (except for 129..256 Grams: the 2 x 2 block path, see
    _chol_inv_2x2, reads its breakdown flags once).  ``defer``: no host
    read on the 2 x 2 path either; its breakdown shows in info[1] and, for
    a shifted mode, the caller re-runs with ``single`` (the one-kernel
    factorisation with the shift schedule)."""
    W = W.contiguous()
    l = W.shape[0]
    if chol_blocked(l) and not single:
        r = _chol_inv_2x2(W, defer=defer)
        if r is not None:
            return r[0], (r[1] if want_inv else None), r[2], r[3]
    Cm = torch.empty_like(W)
    Ci = torch.empty_like(W) if want_inv else None
    nu = _empty(1, like=W)
    info = torch.zeros(2, dtype=torch.int32, device=W.device)
    nw = int(_lib.lib().edak_chol_inv_work_doubles(l))
    work = _empty(nw, like=W) if nw else None
    _lib.call("edak_chol_inv", W.data_ptr(), l, Cm.data_ptr(), _lib.ptr(Ci), int(mode),
              float(scale), nu.data_ptr(), info.data_ptr(), _lib.ptr(work), _lib.stream())
    return Cm, Ci, nu, info


def trinv_upper(R):
    R = R.contiguous()
    X = torch.empty_like(R)
    _lib.call("edak_trinv_upper", R.data_ptr(), R.shape[0], X.data_ptr(), _lib.stream())
    return X


def svd_jacobi(M, want_v=False):
    """One-sided Jacobi SVD of a column block M (cols, rows), rows >= cols:
    returns U (cols, rows) block, sig (cols,) descending, V (cols, cols)."""
    M = M.contiguous()
    cols, rows = M.shape
    U = torch.empty_like(M)
    sig = _empty(cols, like=M)
    V = _empty(cols, cols, like=M) if want_v else None
    work = _empty(int(_lib.lib().edak_svd_work_doubles(rows, cols)), like=M)
    _lib.call("edak_svd_jacobi", M.data_ptr(), rows, cols, U.data_ptr(), sig.data_ptr(),
              _lib.ptr(V), work.data_ptr(), _lib.stream())
    _LAST_SVD[0] = work  # diagnostics: work[-1] = sweeps of the last call (last_svd_sweeps)
    return U, sig, V


_LAST_SVD = [None]


def last_svd_sweeps():
    """Jacobi sweeps of the most recent svd_jacobi call (synchronises)."""
    w = _LAST_SVD[0]
    return None if w is None else int(w[-1].item())
