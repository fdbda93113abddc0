"""Pins of the probe -> symbol assembly oracle (SPEC.md:296-367 examples as test ideas).

Checked against closed forms and brute force, never against itself: identity operator (symbol == 1), an exact
Fourier multiplier (rows == multiplier), an exact spatial multiplier (columns == multiplier), the product-
convolution identity with explicit correlation sums, partition of unity / interpolation of the weights,
trigonometric exactness of the angular interpolant, and batching soundness for an exactly local operator."""
import math

import numpy as np
import pytest

from oracle import probing as pr
from oracle import psido


def fourier_multiplier(q):
    return lambda v: np.real(np.fft.ifft2(q * np.fft.fft2(v)))


def test_psf_identity_rows_are_one():
    nz, nx = 24, 30
    pts = [(6, 7), (6, 22), (17, 7), (17, 22)]
    batch = [0, 1, 1, 0]
    P = pr.delta_probes(nz, nx, pts, batch)
    rows = pr.psf_symbol_rows(pr.extract_psfs(P, pts, batch, radius=3))
    assert np.max(np.abs(rows - 1.0)) < 1e-12


def test_psf_rows_recover_fourier_multiplier():
    """H = multiplier q(xi) = 1 + 0.3 cos(xi_x h) + 0.2 cos(xi_z h) (kernel support radius 1):
    every symbol row equals q exactly."""
    nz, nx, h = 20, 28, 1.0
    fz = 2 * math.pi * np.fft.fftfreq(nz, d=h)
    fx = 2 * math.pi * np.fft.fftfreq(nx, d=h)
    q = 1 + 0.3 * np.cos(fx[None, :] * h) + 0.2 * np.cos(fz[:, None] * h)
    H = fourier_multiplier(q)
    pts = [(5, 5), (14, 20)]
    P = pr.delta_probes(nz, nx, pts, [0, 0])
    R = np.stack([H(p) for p in P])
    rows = pr.psf_symbol_rows(pr.extract_psfs(R, pts, [0, 0], radius=2))
    for k in range(2):
        assert np.max(np.abs(rows[k] - q)) < 1e-12


def test_product_convolution_identity_brute_force():
    """psido.apply(w, rows, v)(x) = sum_k w_k(x) sum_z p_k(z) v(x + z) (periodic), written as explicit sums."""
    rng = np.random.default_rng(0)
    nz, nx, rad = 9, 11, 2
    pts = [(2, 3), (6, 8)]
    R = rng.standard_normal((2, nz, nx))
    psfs = pr.extract_psfs(R, pts, [0, 1], rad)
    rows = pr.psf_symbol_rows(psfs)
    w = pr.psf_weights(nz, nx, [2, 6], [3, 8])[[0, 3]]
    v = rng.standard_normal((nz, nx))
    out = psido.apply(w, rows, v)
    ref = np.zeros((nz, nx))
    for k in range(2):
        for z in range(nz):
            for x in range(nx):
                acc = 0.0
                for dz in range(-rad, rad + 1):
                    for dx in range(-rad, rad + 1):
                        acc += psfs[k, dz % nz, dx % nx] * v[(z + dz) % nz, (x + dx) % nx]
                ref[z, x] += w[k, z, x] * acc
    assert np.max(np.abs(out - ref)) < 1e-12


def test_psf_weights_partition_and_interpolation():
    nz, nx = 30, 41
    lz, lx = [4, 13, 25], [3, 20, 37]
    w = pr.psf_weights(nz, nx, lz, lx)
    assert np.max(np.abs(w.sum(0) - 1.0)) < 1e-12
    assert np.all(w >= -1e-15)
    for i, z in enumerate(lz):
        for j, x in enumerate(lx):
            k = i * len(lx) + j
            e = np.zeros(len(lz) * len(lx))
            e[k] = 1.0
            assert np.allclose(w[:, z, x], e, atol=1e-14)
    w2 = pr.psf_weights(1, 21, [0], [4, 14])     # two points, midpoint x = 9 -> 0.5 / 0.5
    assert abs(w2[0, 0, 9] - 0.5) < 1e-14 and abs(w2[1, 0, 9] - 0.5) < 1e-14


def test_batching_soundness_local_operator():
    """For an operator that is exactly local within the window (variable-coefficient 5-point stencil), PSFs from
    batched probes equal PSFs from one-point-per-probe runs."""
    rng = np.random.default_rng(1)
    nz, nx = 26, 26
    a = 1 + 0.5 * rng.random((nz, nx))

    def H(v):
        lap = -4 * v + np.roll(v, 1, 0) + np.roll(v, -1, 0) + np.roll(v, 1, 1) + np.roll(v, -1, 1)
        return a * v + 0.3 * lap
    pts = [(4, 4), (4, 13), (13, 4), (13, 13), (21, 21)]
    batched = [0, 1, 1, 0, 0]
    single = list(range(5))
    Rb = np.stack([H(p) for p in pr.delta_probes(nz, nx, pts, batched)])
    Rs = np.stack([H(p) for p in pr.delta_probes(nz, nx, pts, single)])
    pb = pr.extract_psfs(Rb, pts, batched, radius=3)
    ps = pr.extract_psfs(Rs, pts, single, radius=3)
    assert np.max(np.abs(pb - ps)) < 1e-12


def test_pdo_plan_antipodal_and_probe_real():
    idx, th = pr.pdo_plan(64, 64, 10.0, rho0=2 * math.pi * 0.02, r=8)
    assert len(idx) == 8
    for k in range(4):
        a, b = idx[k], idx[k + 4]
        assert ((a[0] + b[0]) % 64, (a[1] + b[1]) % 64) == (0, 0)
    v = pr.sinusoid_probe(64, 64, idx)
    assert np.max(np.abs(v.imag)) < 1e-12
    spec = np.abs(np.fft.fft2(v.real))
    assert np.count_nonzero(spec > 1e-6 * spec.max()) == len(set(idx))


def test_pdo_identity_columns_are_one():
    nz, nx, h = 64, 64, 10.0
    idx, th = pr.pdo_plan(nz, nx, h, rho0=2 * math.pi * 0.02, r=8)
    v = pr.sinusoid_probe(nz, nx, idx).real
    cols = pr.extract_symbol_columns(v, idx, mask_radius=3.0)
    assert np.max(np.abs(cols - 1.0)) < 1e-10


def test_pdo_columns_recover_spatial_multiplier():
    """H = D_a with a band-limited a (spectrum inside the mask disc): every column equals a."""
    nz, nx, h = 64, 64, 10.0
    iz = np.arange(nz)[:, None]
    ix = np.arange(nx)[None, :]
    a = 2.0 + 0.4 * np.cos(2 * math.pi * 2 * ix / nx) + 0.3 * np.sin(2 * math.pi * 1 * iz / nz)
    idx, th = pr.pdo_plan(nz, nx, h, rho0=2 * math.pi * 0.025, r=8)
    v = pr.sinusoid_probe(nz, nx, idx).real
    cols = pr.extract_symbol_columns(a * v, idx, mask_radius=3.0)
    assert np.max(np.abs(cols - a)) < 1e-10


def test_dirichlet_weights():
    r = 8
    th = np.array([2 * math.pi * k / r for k in range(1, r + 1)])
    T = pr.dirichlet_kernel(th[:, None] - th[None, :], r)
    assert np.max(np.abs(T - np.eye(r))) < 1e-12
    phis = np.linspace(0, 2 * math.pi, 97)
    f = np.cos(2 * phis)
    interp = sum(np.cos(2 * th[k]) * pr.dirichlet_kernel(phis - th[k], r) for k in range(r))
    assert np.max(np.abs(interp - f)) < 1e-12           # degree 2 < r/2: exact
    nz, nx, h, rho0 = 32, 32, 1.0, 2 * math.pi * 4 / 32
    W = pr.pdo_weights(nz, nx, h, rho0, list(th))
    assert np.all(W[:, 0, 0] == 0.0)                     # value at xi = 0
    # radius 2 rho0 at angle theta_k = pi (k = 4 -> -x direction): w = 2 there
    kx = (-8) % nx
    assert abs(W[3, 0, kx] - 2.0) < 1e-12 and np.max(np.abs(np.delete(W[:, 0, kx], 3))) < 1e-12
