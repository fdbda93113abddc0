"""GPU parity of probe -> symbol assembly against the fp64 oracle, on synthetic responses
and end to end on real H·v responses: PSF rows from spike H·v on the cfg 0 model and PDO columns from a cosine-sum
probe, assembled and applied through hv_psido_apply."""
import math

import numpy as np
import pytest

from oracle import probing as opr
from oracle import psido as opsido
from tests.conftest import rel_l2
import workloads as W

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def hv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_10804_b200 as hvmod
    return hvmod


@pytest.fixture(scope="module")
def solver(hv):
    return hv.Solver.from_workload(W.config(0))


def test_psf_rows_weights_parity(solver):
    rng = np.random.default_rng(0)
    nz, nx = 50, 70
    pts = [(10, 12), (10, 45), (35, 12), (35, 45), (22, 60)]
    batch = [0, 1, 1, 0, 2]
    R = rng.standard_normal((3, nz, nx)).astype(np.float32)
    rows = solver.psf_rows(R, pts, batch, radius=6)
    ref = opr.psf_symbol_rows(opr.extract_psfs(R.astype(np.float64), pts, batch, 6))
    assert rel_l2(rows, ref) <= TOL
    w = solver.psf_weights(nz, nx, [10, 35], [12, 45])
    wref = opr.psf_weights(nz, nx, [10, 35], [12, 45])
    assert np.max(np.abs(w - wref)) <= 1e-6


def test_pdo_columns_weights_parity(solver):
    rng = np.random.default_rng(1)
    nz, nx, h = 64, 96, 8.0
    idx, th = opr.pdo_plan(nz, nx, h, rho0=2 * math.pi * 0.02, r=8)
    R = rng.standard_normal((nz, nx)).astype(np.float32)
    cols = solver.pdo_columns(R, idx, mask_radius=3.0)
    ref = opr.extract_symbol_columns(R.astype(np.float64), idx, 3.0)
    assert rel_l2(cols, ref) <= TOL
    w = solver.pdo_weights(nz, nx, h, 2 * math.pi * 0.02, th)
    wref = opr.pdo_weights(nz, nx, h, 2 * math.pi * 0.02, th)
    assert rel_l2(w, wref) <= TOL and np.max(np.abs(w.imag)) == 0.0


def _cfg0_spikes():
    """cfg 0 grid and acquisition with 4 PSF spikes on a 2 x 2 lattice (each side computes its own H·v)."""
    wl = W.config(0)
    pts = [(20, 20), (20, 44), (44, 20), (44, 44)]
    V = np.stack([W.spike_probe((64, 64), *p) for p in pts])
    return wl, pts, V


@pytest.fixture(scope="module")
def cfg0_psf_oracle():
    from oracle import wave
    wl, pts, V = _cfg0_spikes()
    HV = wave.Problem(wl).hessvec(list(V.astype(np.float64)))
    rows = opr.psf_symbol_rows(opr.extract_psfs(HV, pts, [0, 1, 2, 3], 12))
    w = opr.psf_weights(64, 64, [20, 44], [20, 44])
    return wl, pts, V, HV, rows, w


@pytest.fixture(scope="module")
def cfg0_pdo_oracle():
    from oracle import wave
    wl = W.config(0)
    rho0 = 2 * math.pi * 0.0125
    idx, th = opr.pdo_plan(64, 64, wl.h, rho0, r=8)
    vp = opr.sinusoid_probe(64, 64, idx).real.astype(np.float32)
    R = wave.Problem(wl).hessvec([vp.astype(np.float64)])[0]
    cols = opr.extract_symbol_columns(R, idx, 2.5)
    wts = opr.pdo_weights(64, 64, wl.h, rho0, th)
    return wl, rho0, idx, th, vp, cols, wts


def test_psf_pipeline_end_to_end(hv, cfg0_psf_oracle):
    """H·v on 4 spikes -> rows -> hat weights -> apply_psf, each side from its own H·v."""
    wl, pts, V, HV_ref, rows_ref, w_ref = cfg0_psf_oracle
    s = hv.Solver.from_workload(wl)
    HV = s.hessvec(wl.model, V)
    rows = s.psf_rows(HV, pts, [0, 1, 2, 3], radius=12)
    assert rel_l2(rows, rows_ref) <= TOL
    w = s.psf_weights(64, 64, [20, 44], [20, 44])
    v = W.gaussian_probe((64, 64), 5, 3.0)
    out = s.psido_apply(w, rows, v, 0)
    ref = opsido.apply(w_ref, rows_ref, v.astype(np.float64))
    assert rel_l2(out, ref) <= TOL


def test_pdo_pipeline_end_to_end(hv, cfg0_pdo_oracle):
    """H·v on the 8-angle cosine-sum probe -> columns -> weights -> apply_pdo (symmetrised)."""
    wl, rho0, idx, th, vp, cref, wref = cfg0_pdo_oracle
    s = hv.Solver.from_workload(wl)
    R = s.hessvec(wl.model, vp[None])[0]
    cols = s.pdo_columns(R, idx, mask_radius=2.5)
    assert rel_l2(cols, cref) <= TOL
    w = s.pdo_weights(64, 64, wl.h, rho0, th)
    v = W.gaussian_probe((64, 64), 9, 3.0)
    out = s.psido_apply(np.ascontiguousarray(cols.real), w, v, 2)
    ref = opsido.apply_symmetric(cref.real, wref, v.astype(np.float64))
    assert rel_l2(out, ref) <= TOL


def test_psf_plus_synthetic_parity(solver):
    from oracle import psfplus as opp
    rng = np.random.default_rng(4)
    nz, nx, nr, nc, rank = 24, 32, 6, 4, 3
    N = nz * nx
    Bt = np.linalg.qr(rng.standard_normal((N, 4)) + 1j * rng.standard_normal((N, 4)))[0].T
    rows = ((rng.standard_normal((nr, 4)) + 1j * rng.standard_normal((nr, 4))) @ Bt).reshape(nr, nz, nx)
    rows = (rows + 1e-3 * (rng.standard_normal(rows.shape) + 1j * rng.standard_normal(rows.shape))).astype(np.complex64)
    w = rng.random((nr, nz, nx)).astype(np.float32)
    cols = (rng.standard_normal((nc, nz, nx)) + 1j * rng.standard_normal((nc, nz, nx))).astype(np.complex64)
    idx = [(1, 2), (3, 7), (5, 1), (20, 30)]
    A, B, alpha = solver.psf_plus(rows, w, cols, idx, rank)
    Ar, Br, aref = opp.psf_plus(rows.astype(np.complex128), w.astype(np.float64), cols.astype(np.complex128), idx, rank)
    assert abs(alpha - aref) <= 1e-5 * aref
    v = rng.standard_normal((nz, nx)).astype(np.float32)
    out = solver.psido_apply(A, B, v, 0)
    ref = opp.apply(Ar, Br, v.astype(np.float64))
    assert rel_l2(out, ref) <= TOL
    # the factorisation is unique up to per-column phases: compare the symbol A B at sampled (x, xi)
    S = np.einsum("kx,ky->xy", A.reshape(rank, N)[:, ::97], B.reshape(rank, N)[:, ::89])
    Sr = np.einsum("xk,ky->xy", Ar[::97], Br[:, ::89])
    assert rel_l2(S, Sr) <= TOL


def test_psf_plus_pipeline_end_to_end(hv, cfg0_psf_oracle, cfg0_pdo_oracle):
    """PSF rows + PDO columns of the cfg 0 H_d (each side from its own H·v) -> PSF+ rank 3 -> apply."""
    from oracle import psfplus as opp
    wl, pts, V, HV_ref, rows_ref, w_ref = cfg0_psf_oracle
    _, rho0, idx, th, vp, cref, wref = cfg0_pdo_oracle
    s = hv.Solver.from_workload(wl)
    HV = s.hessvec(wl.model, V)
    rows = s.psf_rows(HV, pts, [0, 1, 2, 3], radius=12)
    w = s.psf_weights(64, 64, [20, 44], [20, 44])
    R = s.hessvec(wl.model, vp[None])[0]
    cols = s.pdo_columns(R, idx, mask_radius=2.5)
    A, B, alpha = s.psf_plus(rows, w, cols, idx, 3)
    Ar, Br, aref = opp.psf_plus(rows_ref, w_ref, cref, idx, 3)
    assert abs(alpha - aref) <= 1e-4 * aref
    v = W.gaussian_probe((64, 64), 13, 3.0)
    assert rel_l2(s.psido_apply(A, B, v, 0), opp.apply(Ar, Br, v.astype(np.float64))) <= TOL


def test_highpass_parity_and_wrapped_hessian(hv):
    from oracle import highpass as ohp
    from oracle import wave
    rng = np.random.default_rng(3)
    V = rng.standard_normal((3, 40, 56)).astype(np.float32)
    s = hv.Solver.from_workload(W.config(0))
    out = s.highpass(V, 10.0, 0.05, 0.03)
    assert rel_l2(out, ohp.apply(V.astype(np.float64), 10.0, 0.05, 0.03)) <= TOL
    # wrapped operator Q H Q on cfg 0 against the oracle's Q H Q (and it stays symmetric)
    wl = W.config(0)
    P = np.stack([wl.probe_fn(0), W.gaussian_probe((64, 64), 11, 2.0)])
    got = s.hessvec_highpass(wl.model, P, wl.h, 0.02, 0.01)
    ref = ohp.wrap(lambda X: wave.Problem(wl).hessvec(list(X)), wl.h, 0.02, 0.01)(P.astype(np.float64))
    assert rel_l2(got, ref) <= TOL
    a, b = float(np.sum(P[1] * got[0])), float(np.sum(P[0] * got[1]))
    assert abs(a - b) <= 1e-4 * max(abs(a), abs(b))


def test_lowrank_geneig_parity_cfg0(hv):
    """N2: randomized generalized eigensolver on the cfg 0 H_d with the same Omega on both sides."""
    from oracle import lowrank as olr
    from oracle import wave
    wl = W.config(0)
    K, r, q = 12, 6, 1
    Om = np.stack([W.gaussian_probe((64, 64), 100 + k, 1.0) for k in range(K)])
    delta, gamma = 1.0, 4.0 * wl.h ** 2
    s = hv.Solver.from_workload(wl)
    ev, V = s.lowrank_geneig(wl.model, Om, r, power_iters=q, delta=delta, gamma=gamma)
    pb = wave.Problem(wl)
    lam, Vr = olr.randomized_gen_eig(lambda X: pb.hessvec(list(X)), Om.astype(np.float64), r, q, wl.h, delta, gamma)
    assert np.all(np.diff(ev) <= 0)
    assert np.max(np.abs(ev - lam) / lam[0]) <= 1e-4, (ev, lam)
    RV = olr.prior_apply(Vr, wl.h, delta, gamma)
    for i in range(r):
        gap = min(abs(lam[i] - lam[j]) for j in range(r) if j != i) / lam[0]
        if gap > 1e-2:
            c = abs(float(np.sum(V[i].astype(np.float64) * RV[i])))
            assert abs(c - 1.0) <= 1e-3, (i, c)
