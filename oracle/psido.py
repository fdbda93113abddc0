"""fp64 oracle of the low-rank-symbol PsiDO apply (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

PAPER.md:240-247 (Eqs. equ:lr_symbol, equ:lr-psido): s(x, xi) ~ sum_k a_k(x) b_k(xi) and
    H_d ~ sum_{k=1..r} D_{a_k} F^{-1} D_{b_k} F,
"one Fourier transform, r inverse Fourier transforms, and 2r pointwise multiplications".

Discrete reading: F = unnormalised 2-D DFT on the interior
grid [nz][nx] with unshifted frequency order, F^{-1} = its exact inverse (1/N). This equals
SPEC.md's scaled pair: dx dz/(2 pi)^2 times (2 pi)^2/(dx dz N) = 1/N.
a_k real, b_k complex; the real part of the result is returned (real-in/real-out).
Adjoint under the Euclidean inner product: sum_k Re F^{-1}(conj(b_k) . F(a_k . v));
symmetric = (apply + adjoint)/2.
"""
from __future__ import annotations

import numpy as np


def apply(a: np.ndarray, b: np.ndarray, v: np.ndarray) -> np.ndarray:
    """out = Re sum_k a_k . IDFT(b_k . DFT(v)). a [r][nz][nx] real, b [r][nz][nx] complex, v [nz][nx]."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.complex128)
    vh = np.fft.fft2(np.asarray(v, dtype=np.float64))          # the one forward transform
    out = np.zeros(v.shape)
    for k in range(a.shape[0]):                                   # r inverse transforms
        out += a[k] * np.real(np.fft.ifft2(b[k] * vh))
    return out


def apply_adjoint(a: np.ndarray, b: np.ndarray, v: np.ndarray) -> np.ndarray:
    """out = Re sum_k IDFT(conj(b_k) . DFT(a_k . v))."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.complex128)
    v = np.asarray(v, dtype=np.float64)
    out = np.zeros(v.shape)
    for k in range(a.shape[0]):
        out += np.real(np.fft.ifft2(np.conj(b[k]) * np.fft.fft2(a[k] * v)))
    return out


def apply_symmetric(a: np.ndarray, b: np.ndarray, v: np.ndarray) -> np.ndarray:
    """(apply + apply_adjoint) / 2."""
    return 0.5 * (apply(a, b, v) + apply_adjoint(a, b, v))


def apply_mode(a, b, v, mode: int) -> np.ndarray:
    return (apply, apply_adjoint, apply_symmetric)[mode](a, b, v)
