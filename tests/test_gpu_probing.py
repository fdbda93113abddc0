"""GPU parity of probe -> symbol assembly against the fp64 oracle, on synthetic responses
and end to end on real H·v responses: PSF rows from the cfg 1 spike H·v and PDO columns from a cosine-sum
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


def test_psf_pipeline_on_hessvec_cfg1(hv):
    """End to end on the bench workload's probes (cfg 1, 2 shots to keep the oracle cheap is not needed: the
    pipeline input is the GPU's own H·v, and each stage is checked against the oracle applied to the same
    input): H·v on 4 spikes -> rows -> hat weights -> apply_psf on a smooth probe."""
    wl = W.config(1).subset(shots=[3, 12])
    ks = [2 * 8 + 2, 2 * 8 + 5, 5 * 8 + 2, 5 * 8 + 5]
    V = wl.probes(ks)
    s = hv.Solver.from_workload(wl)
    HV = s.hessvec(wl.model, V)
    pts = [tuple(int(c) for c in np.argwhere(v)[0]) for v in V]
    rows = s.psf_rows(HV, pts, [0, 1, 2, 3], radius=20)
    rows_ref = opr.psf_symbol_rows(opr.extract_psfs(HV.astype(np.float64), pts, [0, 1, 2, 3], 20))
    assert rel_l2(rows, rows_ref) <= TOL
    lz = sorted({p[0] for p in pts})
    lx = sorted({p[1] for p in pts})
    w = s.psf_weights(wl.nz, wl.nx, lz, lx)
    v = W.gaussian_probe((wl.nz, wl.nx), 5, 4.0)
    out = s.psido_apply(w, rows, v, 0)
    ref = opsido.apply(opr.psf_weights(wl.nz, wl.nx, lz, lx), rows_ref, v.astype(np.float64))
    assert rel_l2(out, ref) <= TOL


def test_pdo_pipeline_on_hessvec_cfg1(hv):
    """H·v on the cosine-sum probe of an 8-angle plan -> columns -> weights -> apply_pdo."""
    wl = W.config(1).subset(shots=[7])
    rho0 = 2 * math.pi * 0.012
    idx, th = opr.pdo_plan(wl.nz, wl.nx, wl.h, rho0, r=8)
    vp = opr.sinusoid_probe(wl.nz, wl.nx, idx).real.astype(np.float32)
    s = hv.Solver.from_workload(wl)
    R = s.hessvec(wl.model, vp[None])[0]
    cols = s.pdo_columns(R, idx, mask_radius=4.0)
    cref = opr.extract_symbol_columns(R.astype(np.float64), idx, 4.0)
    assert rel_l2(cols, cref) <= TOL
    w = s.pdo_weights(wl.nz, wl.nx, wl.h, rho0, th)
    a = np.ascontiguousarray(cols.real)
    v = W.gaussian_probe((wl.nz, wl.nx), 9, 3.0)
    out = s.psido_apply(a, w, v, 2)
    ref = opsido.apply_symmetric(cref.real, opr.pdo_weights(wl.nz, wl.nx, wl.h, rho0, th), v.astype(np.float64))
    assert rel_l2(out, ref) <= TOL


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
