"""fp64 oracle of the high-pass wrapper, SURVEY.md §8(f) N4 (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PAPER.md:200 / 361 (§3.7): "we apply a high-pass filter to H_d before the approximation, removing low-frequency
components". The filter is the Fourier multiplier Q = IDFT diag(q) DFT (SPEC.md:267-270, 377-384 reading):
q(xi) = 0 for |xi| <= xi_c - w/2, 1 for |xi| >= xi_c + w/2, raised cosine in between; wrapped operator Q H Q.
Frequencies: unshifted DFT order on the interior grid with spacing h (DESIGN.md §3 R-highpass).
"""
from __future__ import annotations

import math

import numpy as np


def multiplier(nz: int, nx: int, h: float, cutoff: float, width: float) -> np.ndarray:
    fz = 2 * math.pi * np.fft.fftfreq(nz, d=h)
    fx = 2 * math.pi * np.fft.fftfreq(nx, d=h)
    rho = np.sqrt(fz[:, None] ** 2 + fx[None, :] ** 2)
    lo, hi = cutoff - width / 2.0, cutoff + width / 2.0
    q = np.where(rho >= hi, 1.0, 0.0)
    band = (rho > lo) & (rho < hi)
    q[band] = 0.5 * (1.0 - np.cos(math.pi * (rho[band] - lo) / width))
    return q


def apply(v: np.ndarray, h: float, cutoff: float, width: float) -> np.ndarray:
    """Q v for v [..][nz][nx]."""
    v = np.asarray(v, dtype=np.float64)
    q = multiplier(v.shape[-2], v.shape[-1], h, cutoff, width)
    return np.real(np.fft.ifft2(q * np.fft.fft2(v)))


def wrap(H, h: float, cutoff: float, width: float):
    """v -> Q H Q v."""
    return lambda V: apply(H(apply(V, h, cutoff, width)), h, cutoff, width)
