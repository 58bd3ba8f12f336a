"""Background/observation covariances (mirrors reference ``covariance.py``).

``GridCovFactor`` / ``DiagonalNoise`` keep the reference constructors and
duck type (``.n``, ``.symbol``, ``.apply``, ``.apply_t``; ``.sigma``,
``.apply``, ``.solve``; covariance.py:22-71).  ``apply`` runs the sm_100a
circulant kernel (``edak_circ_apply``) instead of numpy's FFT.

``gaussian_factor`` is the BASELINE configs' Gaussian correlation
C_ij = exp(-d_ij^2 / (2 L^2)) with B^{1/2} the circulant square root from the
DFT of C's first row, evaluated in closed form (Poisson summation) so that
every eigenvalue is positive and exact to a few ulp.

``factor_taps(ub)`` turns ANY symmetric circulant factor with a ``.symbol``
(ours or the reference's GridCovFactor) into the device tap list the
kernels take: the generator u = irfft(symbol) truncated where |u_d| falls
below 1e-15 max|u| (the Gaussian generator decays like exp(-d^2/L^2):
97 / 189 / 377 taps at L = 8 / 16 / 32; measured conv-vs-FFT error
<= 7e-16 relative), or all n taps when the band would cover the ring.
"""

import numpy as np
import torch

from . import _dev, _lib

TAP_TOL = 1e-15
MAX_TAPS = 4096


class CirculantFactor:
    """Symmetric circulant U_B given by the rfft half of its symbol."""

    def __init__(self, n, symbol, sigma_b=None):
        self.n = int(n)
        self.symbol = np.asarray(symbol, dtype=float)
        if self.symbol.shape != (self.n // 2 + 1,):
            raise ValueError("symbol must have n // 2 + 1 entries")
        self.sigma_b = sigma_b

    def apply(self, v):
        """U_B v for (n,) or (n, l) numpy / torch input (covariance.py:41-45)."""
        return apply_factor(self, v)

    apply_t = apply  # symmetric factor (covariance.py:47)

    def correlation(self):
        s = 1.0 if self.sigma_b is None else self.sigma_b
        return np.fft.irfft(self.symbol ** 2, n=self.n) / s ** 2

    def dense(self):
        """The factor as an (n, n) host matrix, small n only (covariance.py:53-56):
        entry (i, j) is the generator at (i - j) mod n."""
        u = np.fft.irfft(self.symbol, n=self.n)
        i = np.arange(self.n)
        return u[(i[:, None] - i[None, :]) % self.n]


class GridCovFactor(CirculantFactor):
    """Reference diffusion-spectrum factor (covariance.py:22-39): symbol
    u(m) = sigma_b gamma (1 + 4 kappa sin^2(pi m / n))^-M, kappa = D^2/(4M)."""

    def __init__(self, n, sigma_b, length_scale, n_passes):
        kappa = length_scale ** 2 / (4.0 * n_passes)
        m = np.arange(n)
        shape = (1.0 + 4.0 * kappa * np.sin(np.pi * m / n) ** 2) ** (-n_passes)
        gamma = np.sqrt(n / np.sum(shape ** 2))
        super().__init__(n, (sigma_b * gamma * shape)[: n // 2 + 1], sigma_b)
        self.length_scale = length_scale
        self.n_passes = n_passes


def gaussian_spectrum(n, length):
    """Closed-form DFT of the periodic Gaussian correlation row (all > 0)."""
    m = np.arange(n // 2 + 1, dtype=float) / n
    c = np.zeros_like(m)
    for k in range(-3, 4):
        c += np.exp(-2.0 * np.pi ** 2 * length ** 2 * (m - k) ** 2)
    return np.sqrt(2.0 * np.pi) * length * c


def gaussian_factor(n, sigma_b, length):
    """U_B = sigma_b C^{1/2}, C_ij = exp(-d_ij^2 / (2 L^2))."""
    return CirculantFactor(n, sigma_b * np.sqrt(gaussian_spectrum(n, length)), sigma_b)


class DiagonalNoise:
    """R = sigma^2 I (covariance.py:59-71)."""

    def __init__(self, sigma):
        self.sigma = sigma

    def apply(self, w):
        return self.sigma * w

    def solve(self, w):
        return w / self.sigma ** 2


def factor_taps(ub):
    """(taps, tap_w) host arrays for any factor exposing ``.n``/``.symbol``."""
    n = int(ub.n)
    u = np.fft.irfft(np.asarray(ub.symbol, dtype=float), n=n)
    a = np.abs(u)
    d = np.minimum(np.arange(n), n - np.arange(n))
    big = a > TAP_TOL * a.max() if a.max() > 0 else np.zeros(n, bool)
    w = int(d[big].max()) if big.any() else 0
    if 2 * w + 1 >= n:
        k = n
        w = (n - 1) // 2
    else:
        k = 2 * w + 1
    if k > MAX_TAPS:
        raise ValueError(f"circulant factor needs {k} taps (> {MAX_TAPS}); "
                         "its generator does not decay on this ring")
    taps = u[(np.arange(k) - w) % n]
    return np.ascontiguousarray(taps), w


def os_tables(taps, w, logm):
    """Overlap-save tables for circ_os.cu: the block kernel
    h[m mod M] = taps[m + w] (m = k - w, k < K), its spectrum fft(h) / M in
    bit-reversed order (the forward DIF's output order), and the twiddles
    exp(-2 pi i m / (2M)), m < M -- both as interleaved (re, im) float64."""
    M = 1 << logm
    h = np.zeros(M)
    k = np.arange(taps.size)
    np.add.at(h, (k - w) % M, taps)
    H = np.fft.fft(h) / M
    rev = np.array([int(format(j, f"0{logm}b")[::-1], 2) for j in range(M)])
    Hr = H[rev]
    spec = np.empty(2 * M)
    spec[0::2], spec[1::2] = Hr.real, Hr.imag
    ang = np.pi * (np.arange(M, dtype=float) / M)  # m / M exact for power-of-two M
    tw = np.empty(2 * M)
    tw[0::2], tw[1::2] = np.cos(ang), -np.sin(ang)
    return spec, tw


def os_logm_for(n, ntaps):
    """Block size (log2) of the overlap-save U_B, or 0 for the tap
    convolution: blocks of M = 1024 (K <= 256) or 2048 (K <= 512) complex
    points on rings of at least 4096 points with a genuinely banded factor."""
    if n < 4096 or 2 * ntaps > n:
        return 0
    if ntaps <= 256:
        return 10
    if ntaps <= 512:
        return 11
    return 0


class DeviceFactor:
    """Device-resident taps (and, on long rings, the overlap-save block
    spectrum + twiddles) of a circulant factor, plus a minimal edak_problem
    that the U_B kernels read."""

    def __init__(self, ub):
        self.n = int(ub.n)
        taps, w = factor_taps(ub)
        self.taps = _dev.f64(taps)
        self.tap_w = w
        self.ntaps = taps.size
        n = self.n
        self.os_spec = self.os_tw = None
        self.os_logm = os_logm_for(n, self.ntaps)
        if self.os_logm:
            spec, tw = os_tables(taps, w, self.os_logm)
            self.os_spec, self.os_tw = _dev.f64(spec), _dev.f64(tw)
        self._prob = _lib.Problem()
        self._prob.n = self.n
        self._prob.taps = self.taps.data_ptr()
        self._prob.ntaps = self.ntaps
        self._prob.tap_w = w
        self._prob.os_spec, self._prob.os_tw = _lib.ptr(self.os_spec), _lib.ptr(self.os_tw)
        self._prob.os_logm = self.os_logm

    def apply_cols(self, cols, out=None):
        """U_B applied to a (ncols, n) device block."""
        cols = cols.contiguous()
        out = torch.empty_like(cols) if out is None else out
        _lib.call("edak_circ_apply", _lib.C.byref(self._prob), cols.data_ptr(),
                  out.data_ptr(), cols.shape[0], _lib.stream())
        return out


_FACTORS = {}


def device_factor(ub):
    """Cached DeviceFactor for a factor object (keyed by identity+symbol)."""
    key = (id(ub), ub.n)
    df = _FACTORS.get(key)
    if df is None or not np.array_equal(getattr(df, "_symbol", None), ub.symbol):
        df = DeviceFactor(ub)
        df._symbol = np.array(ub.symbol, copy=True)
        _FACTORS[key] = df
    return df


def apply_factor(ub, v):
    cols, vec, as_np = _dev.to_cols(v, ub.n)
    out = device_factor(ub).apply_cols(cols)
    return _dev.from_cols(out, vec, as_np)
