"""Circulant background-covariance factors and the diagonal R (restates
reference ``covariance.py``).

``CirculantFactor`` is the duck type of the reference ``GridCovFactor``
(``.n``, ``.symbol``, ``.apply``, ``.apply_t``; covariance.py:22-56): a
symmetric circulant U_B given by the real-FFT half of its (real, even)
symbol, applied as irfft(symbol * rfft(v)) (covariance.py:41-47).

Two symbol builders:

* ``diffusion_symbol``: the reference's M-pass implicit-diffusion shape
  (covariance.py:29-39).  Used to pin the reference's own fixtures.
* ``gaussian_symbol``: the BASELINE configs' Gaussian correlation
  C_ij = exp(-d_ij^2 / (2 L^2)), d = periodic grid distance, with
  B^{1/2} the circulant square root from the DFT of C's first row.  The
  reference has no Gaussian factor; the DFT is evaluated in
  closed form by Poisson summation,
      c_hat(m) = sqrt(2 pi) L sum_k exp(-2 pi^2 L^2 (m/n - k)^2),
  a sum of positive terms, so every eigenvalue is positive and accurate to
  a few ulp *relative* -- unlike rfft(row), whose tail is rounding noise of
  either sign (|noise| ~ 1e-14) that a sqrt turns into a ~1e-7 symbol floor.
  The closed form equals the DFT of the periodic-distance row up to the
  wrap images exp(-(n/2)^2 / (2 L^2)) (< 1e-21 for every BASELINE config).
  This choice is documented in DESIGN.md ("Gaussian B").
"""

import numpy as np


class CirculantFactor:
    """Symmetric circulant square-root factor U_B (GridCovFactor duck type)."""

    def __init__(self, n, symbol, sigma_b=None):
        self.n = int(n)
        self.symbol = np.asarray(symbol, dtype=float)
        if self.symbol.shape != (self.n // 2 + 1,):
            raise ValueError("symbol must have n // 2 + 1 entries")
        self.sigma_b = sigma_b

    def apply(self, v):
        """U_B v for a vector, or column-wise (axis 0) for a matrix
        (covariance.py:41-45)."""
        vhat = np.fft.rfft(v, axis=0)
        vhat *= self.symbol[:, None] if vhat.ndim == 2 else self.symbol
        return np.fft.irfft(vhat, n=self.n, axis=0)

    apply_t = apply  # symmetric factor (covariance.py:47)

    def first_column(self):
        """Circulant generator u with (U_B v)_i = sum_j u[(i-j) mod n] v_j."""
        return np.fft.irfft(self.symbol, n=self.n)

    def correlation(self):
        """First row of B / sigma_b^2 (covariance.py:49-51)."""
        s = 1.0 if self.sigma_b is None else self.sigma_b
        return np.fft.irfft(self.symbol ** 2, n=self.n) / s ** 2

    def dense(self):
        """Dense U_B (small n; covariance.py:53-56)."""
        u = self.first_column()
        idx = (np.arange(self.n)[:, None] - np.arange(self.n)[None, :]) % self.n
        return u[idx]


def diffusion_symbol(n, sigma_b, length_scale, n_passes):
    """Reference diffusion-spectrum symbol (covariance.py:29-39)."""
    kappa = length_scale ** 2 / (4.0 * n_passes)
    m = np.arange(n)
    shape = (1.0 + 4.0 * kappa * np.sin(np.pi * m / n) ** 2) ** (-n_passes)
    gamma = np.sqrt(n / np.sum(shape ** 2))
    return (sigma_b * gamma * shape)[: n // 2 + 1]


def diffusion_factor(n, sigma_b, length_scale, n_passes):
    """GridCovFactor(n, sigma_b, D, M) restated (covariance.py:22-39)."""
    return CirculantFactor(
        n, diffusion_symbol(n, sigma_b, length_scale, n_passes), sigma_b)


def gaussian_spectrum(n, length):
    """Closed-form DFT of the periodic Gaussian correlation row (see module
    docstring); returns the rfft half, all entries > 0."""
    m = np.arange(n // 2 + 1, dtype=float) / n
    c = np.zeros_like(m)
    for k in range(-3, 4):
        c += np.exp(-2.0 * np.pi ** 2 * length ** 2 * (m - k) ** 2)
    return np.sqrt(2.0 * np.pi) * length * c


def gaussian_factor(n, sigma_b, length):
    """U_B = sigma_b * C^{1/2} for the Gaussian correlation of length L."""
    return CirculantFactor(
        n, sigma_b * np.sqrt(gaussian_spectrum(n, length)), sigma_b)


class DiagonalNoise:
    """R = sigma^2 I (covariance.py:59-71)."""

    def __init__(self, sigma):
        self.sigma = sigma

    def apply(self, w):
        return self.sigma * w

    def solve(self, w):
        return w / self.sigma ** 2
