"""Pins of the PSF+ oracle (N3): the closed-form least squares limits (SPEC.md:369-375 examples), exact
low-rank consistency, the normal equations, and the complex-factor apply against explicit dense sums."""
import math

import numpy as np

from oracle import psfplus as pp


def _setup(rng, nz=8, nx=10, nr=6, true_rank=3, nc=4):
    N = nz * nx
    Bt = np.linalg.qr(rng.standard_normal((N, true_rank)) + 1j * rng.standard_normal((N, true_rank)))[0].T
    coef = rng.standard_normal((nr, true_rank)) + 1j * rng.standard_normal((nr, true_rank))
    rows = (coef @ Bt).reshape(nr, nz, nx)
    W = rng.random((nr, nz, nx))
    idx = [(1, 2), (3, 7), (5, 1), (6, 9)][:nc]
    return rows, W, idx, N


def test_alpha_to_infinity_gives_psf_factor_and_consistency():
    rng = np.random.default_rng(0)
    rows, W, idx, N = _setup(rng)
    cols = rng.standard_normal((4, 8, 10)) + 1j * rng.standard_normal((4, 8, 10))
    A, B, _ = pp.psf_plus(rows, W, cols, idx, 3, alpha=1e12)
    A0, B0, _ = pp.psf_plus(rows, W, cols, idx, 3, alpha=None)
    # A_0 B reproduces S_psf = W rows exactly when the rows have rank 3
    Spsf = W.reshape(6, N).T @ rows.reshape(6, N)
    U, s, Vh = np.linalg.svd(rows.reshape(6, N), full_matrices=False)
    A0 = W.reshape(6, N).T @ (U[:, :3] * s[:3])
    assert np.max(np.abs(A0 @ Vh[:3] - Spsf)) < 1e-10
    assert np.max(np.abs(A - A0)) < 1e-8 * np.max(np.abs(A0))
    # columns consistent with A_0 B at I_c -> A = A_0 for the paper's alpha as well
    ic = [kz * 10 + kx for kz, kx in idx]
    cons = (A0 @ Vh[:3][:, ic]).T.reshape(4, 8, 10)
    A2, _, _ = pp.psf_plus(rows, W, cons, idx, 3)
    assert np.max(np.abs(A2 - A0)) < 1e-10 * np.max(np.abs(A0))


def test_alpha_to_zero_interpolates_columns_and_alpha_rule():
    rng = np.random.default_rng(1)
    rows, W, idx, N = _setup(rng, nc=3)
    cols = rng.standard_normal((3, 8, 10)) + 1j * rng.standard_normal((3, 8, 10))
    A, B, _ = pp.psf_plus(rows, W, cols, idx[:3], 3, alpha=1e-14)
    ic = [kz * 10 + kx for kz, kx in idx[:3]]
    assert np.max(np.abs(A @ B[:, ic] - cols.reshape(3, N).T)) < 1e-8
    _, B1, alpha = pp.psf_plus(rows, W, cols, idx[:3], 3)
    assert abs(alpha - np.linalg.norm(B1[:, ic]) ** 2 / 3.0) < 1e-12       # ||B||_F^2 = rank (orthonormal rows)


def test_normal_equations_hold():
    rng = np.random.default_rng(2)
    rows, W, idx, N = _setup(rng)
    cols = rng.standard_normal((4, 8, 10)) + 1j * rng.standard_normal((4, 8, 10))
    A, B, alpha = pp.psf_plus(rows, W, cols, idx, 3)
    U, s, Vh = np.linalg.svd(rows.reshape(6, N), full_matrices=False)
    A0 = W.reshape(6, N).T @ (U[:, :3] * s[:3])
    ic = [kz * 10 + kx for kz, kx in idx]
    Bc = B[:, ic]
    Sc = cols.reshape(4, N).T
    # gradient of the objective vanishes: (A Bc - Sc) Bc^H + alpha (A - A0_aligned) = 0, with A0 in B's phase
    A0b = A0 @ (Vh[:3] @ B.conj().T)
    g = (A @ Bc - Sc) @ Bc.conj().T + alpha * (A - A0b)
    assert np.max(np.abs(g)) < 1e-10 * max(1.0, np.max(np.abs(A)))


def test_complex_factor_apply_dense():
    rng = np.random.default_rng(3)
    nz, nx, r = 5, 6, 2
    N = nz * nx
    A = rng.standard_normal((N, r)) + 1j * rng.standard_normal((N, r))
    B = rng.standard_normal((r, N)) + 1j * rng.standard_normal((r, N))
    v = rng.standard_normal((nz, nx))
    iz, ix = np.divmod(np.arange(N), nx)
    F = np.exp(-2j * math.pi * (np.outer(iz, iz) / nz + np.outer(ix, ix) / nx))
    M = sum(np.diag(A[:, k]) @ (np.conj(F) / N) @ np.diag(B[k]) @ F for k in range(r))
    assert np.max(np.abs(pp.apply(A, B, v).ravel() - np.real(M @ v.ravel()))) < 1e-12
