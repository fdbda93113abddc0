"""Pins of the randomized generalized eigensolver oracle (N2): the identity and scaled pencils,
a dense generalized eigensolve (scipy.linalg.eigh) on a small operator with a decaying spectrum, and
R-orthonormality / residuals of the returned pairs."""
import numpy as np
import scipy.linalg

from oracle import lowrank as lr


def test_prior_symbol_closed_forms():
    nz, nx, h, d, g = 16, 24, 2.0, 0.7, 0.3
    c = np.full((1, nz, nx), 2.0)
    assert np.allclose(lr.prior_apply(c, h, d, g), d * d * 2.0, atol=1e-12)
    ix = np.arange(nx)[None, :]
    v = np.cos(2 * np.pi * 3 * ix / nx) * np.ones((nz, 1))
    xi = 2 * np.pi * 3 / (nx * h)
    assert np.allclose(lr.prior_apply(v[None], h, d, g)[0], (d + g * xi * xi) ** 2 * v, atol=1e-12)
    rng = np.random.default_rng(0)
    m = rng.standard_normal((2, nz, nx))
    assert np.allclose(lr.prior_apply(lr.prior_apply(m, h, d, g, -1.0), h, d, g, 1.0), m, atol=1e-12)


def test_scaled_pencil_gives_constant_eigenvalues():
    nz, nx, h, d, g = 10, 12, 1.0, 1.0, 0.5
    Hd = lambda V: 3.5 * lr.prior_apply(V, h, d, g)
    Om = np.random.default_rng(1).standard_normal((6, nz, nx))
    lam, V = lr.randomized_gen_eig(Hd, Om, 4, 1, h, d, g)
    assert np.allclose(lam, 3.5, rtol=1e-10)


def test_against_dense_generalized_eigensolve():
    rng = np.random.default_rng(2)
    nz, nx, h, d, g = 8, 9, 1.0, 1.0, 0.4
    N = nz * nx
    U0 = np.linalg.qr(rng.standard_normal((N, N)))[0]
    spec = 10.0 * 0.55 ** np.arange(N)
    Hm = (U0 * spec) @ U0.T
    Hd = lambda V: (V.reshape(len(V), N) @ Hm.T).reshape(V.shape)
    E = np.eye(N).reshape(N, nz, nx)
    Rm = lr.prior_apply(E, h, d, g).reshape(N, N).T
    ref = scipy.linalg.eigh(Hm, Rm, eigvals_only=True)[::-1]
    Om = rng.standard_normal((20, nz, nx))
    lam, V = lr.randomized_gen_eig(Hd, Om, 10, 2, h, d, g)
    assert np.allclose(lam[:8], ref[:8], rtol=1e-6)
    Vf = V.reshape(10, N)
    assert np.max(np.abs(Vf @ Rm @ Vf.T - np.eye(10))) < 1e-8
    for i in range(5):
        res = Hm @ Vf[i] - lam[i] * Rm @ Vf[i]
        assert np.linalg.norm(res) <= 1e-6 * lam[0] * np.linalg.norm(Rm @ Vf[i])
