"""Pins of the PsiDO apply oracle (Eq. equ:lr-psido) — CPU only.

Checked against: the identity symbol (SPEC.md:183 example), a differential-operator symbol
on an exact plane wave (closed form), a brute-force dense materialisation with the DFT
written out as explicit exponential sums (SPEC.md:219-227 pattern), and the adjoint
identity over random symbols (SPEC.md:230 pattern)."""
import math

import numpy as np

from oracle import psido
from tests.conftest import rel_l2


def test_identity_symbol():
    v = np.random.default_rng(0).standard_normal((12, 20))
    a = np.ones((1, 12, 20))
    b = np.ones((1, 12, 20), dtype=complex)
    for mode in range(3):
        assert rel_l2(psido.apply_mode(a, b, v, mode), v) < 1e-14


def test_laplacian_symbol_on_plane_wave():
    """b(xi) = -|xi|^2, a = 1 is the spectral Laplacian: on cos(xi0 . x) it returns -|xi0|^2 cos."""
    nz, nx, h = 16, 24, 5.0
    kz, kx = 3, 5
    iz = np.arange(nz)[:, None]
    ix = np.arange(nx)[None, :]
    v = np.cos(2 * math.pi * (kz * iz / nz + kx * ix / nx))
    xz = 2 * math.pi * np.fft.fftfreq(nz, d=h)
    xx = 2 * math.pi * np.fft.fftfreq(nx, d=h)
    b = -(xz[:, None] ** 2 + xx[None, :] ** 2)[None].astype(complex)
    a = np.ones((1, nz, nx))
    xi2 = (2 * math.pi * kz / (nz * h)) ** 2 + (2 * math.pi * kx / (nx * h)) ** 2
    assert rel_l2(psido.apply(a, b, v), -xi2 * v) < 1e-12


def _dense(a, b, nz, nx):
    """Dense matrix of v -> Re sum_k a_k IDFT(b_k DFT v) with the DFT as explicit sums."""
    N = nz * nx
    iz, ix = np.divmod(np.arange(N), nx)
    # F[p, q] = exp(-2 pi i (kz z / nz + kx x / nx)), p = frequency index, q = space index
    F = np.exp(-2j * math.pi * (np.outer(iz, iz) / nz + np.outer(ix, ix) / nx))
    Finv = np.conj(F) / N
    M = np.zeros((N, N), dtype=complex)
    for k in range(a.shape[0]):
        M += np.diag(a[k].ravel()) @ Finv @ np.diag(b[k].ravel()) @ F
    return np.real(M)


def test_dense_materialisation_and_adjoint():
    rng = np.random.default_rng(3)
    nz, nx, r = 6, 8, 3
    a = rng.standard_normal((r, nz, nx))
    b = rng.standard_normal((r, nz, nx)) + 1j * rng.standard_normal((r, nz, nx))
    M = _dense(a, b, nz, nx)
    v = rng.standard_normal((nz, nx))
    assert rel_l2(psido.apply(a, b, v).ravel(), M @ v.ravel()) < 1e-12
    assert rel_l2(psido.apply_adjoint(a, b, v).ravel(), M.T @ v.ravel()) < 1e-12
    assert rel_l2(psido.apply_symmetric(a, b, v).ravel(), 0.5 * (M + M.T) @ v.ravel()) < 1e-12


def test_adjoint_identity_random_symbols():
    rng = np.random.default_rng(4)
    for _ in range(20):
        nz, nx = rng.integers(8, 33, 2)
        r = int(rng.integers(1, 5))
        a = rng.standard_normal((r, nz, nx))
        b = rng.standard_normal((r, nz, nx)) + 1j * rng.standard_normal((r, nz, nx))
        u, v = rng.standard_normal((2, nz, nx))
        lhs = np.sum(psido.apply(a, b, u) * v)
        rhs = np.sum(u * psido.apply_adjoint(a, b, v))
        assert abs(lhs - rhs) <= 1e-10 * np.sqrt(np.sum(u * u) * np.sum(v * v)) * np.abs(b).max() * np.abs(a).max() * r
