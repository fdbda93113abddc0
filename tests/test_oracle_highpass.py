"""Pins of the high-pass wrapper oracle (N4): closed forms on constants and plane waves, an explicit-sum dense
materialisation of Q, symmetry and band idempotence."""
import math

import numpy as np

from oracle import highpass as hp


def test_constant_removed_and_high_plane_wave_kept():
    nz, nx, h = 32, 48, 10.0
    c = np.full((nz, nx), 3.0)
    assert np.max(np.abs(hp.apply(c, h, 0.05, 0.02))) < 1e-12
    ix = np.arange(nx)[None, :]
    iz = np.arange(nz)[:, None]
    kx, kz = 10, 6                      # |xi| = 2 pi sqrt((10/480)^2 + (6/320)^2) = 0.176 > cutoff + w/2
    v = np.cos(2 * math.pi * (kx * ix / nx + kz * iz / nz))
    assert np.max(np.abs(hp.apply(v, h, 0.05, 0.02) - v)) < 1e-12
    k2 = 1                              # |xi| = 0.013 < cutoff - w/2 -> removed
    w = np.cos(2 * math.pi * k2 * ix / nx) + 0 * iz
    assert np.max(np.abs(hp.apply(w, h, 0.05, 0.02))) < 1e-12


def test_dense_explicit_sums_and_symmetry():
    nz, nx, h = 6, 8, 1.0
    q = hp.multiplier(nz, nx, h, 1.5, 1.0)
    N = nz * nx
    iz, ix = np.divmod(np.arange(N), nx)
    F = np.exp(-2j * math.pi * (np.outer(iz, iz) / nz + np.outer(ix, ix) / nx))
    Q = np.real(np.conj(F).T @ np.diag(q.ravel()) @ F / N)
    rng = np.random.default_rng(0)
    v = rng.standard_normal((nz, nx))
    assert np.max(np.abs(hp.apply(v, h, 1.5, 1.0).ravel() - Q @ v.ravel())) < 1e-12
    assert np.max(np.abs(Q - Q.T)) < 1e-12
    # band idempotence: q in {0, 1} outside the transition band -> Q^2 = Q on those frequencies
    assert np.all((q == 0) | (q == 1) | ((q > 0) & (q < 1)))
    qq = hp.multiplier(64, 64, 1.0, 1.0, 0.5)
    assert np.all(qq >= 0) and np.all(qq <= 1)
