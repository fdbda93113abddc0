"""Pins of the fp64 wave-path oracle — CPU only, marker "not gpu".

Each test checks the oracle against something other than itself: closed forms (polynomial
exactness of the stencil, the 2-D Green's function, travel times), invariants of the exact
discrete adjoint (dot-product test, symmetry, reciprocity), finite differences of the
forward map, and brute force on tiny grids. A plausible slip anywhere (a dropped term,
a wrong sign or index, a transposed operand) fails at least one of them:
- stencil weights / signs          -> test_laplacian_polynomial_exactness, test_green_function
- time-index pairing (C6)          -> test_born_matches_finite_difference, test_adjoint_identity
- imaging weight 2 dt^2 / v        -> test_gradient_fd, test_hessian_is_gradient_derivative
- v^2 injection weight in adjoint  -> test_adjoint_identity, test_reciprocity
- sponge centring                  -> test_adjoint_identity (with sponge), test_reciprocity
"""
import math

import numpy as np
import pytest

from oracle import wave
from tests.conftest import rel_l2
import workloads as wlmod


def tiny(**kw):
    args = dict(nz=12, nx=12, W=6, nt=80, h=10.0, dt=1e-3, ns=2, f_peak=20.0, n_probes=2, seed=3)
    args.update(kw)
    return wlmod.custom(**args)


def edge_free(shape, seed, ring=1):
    """Random interior direction vanishing on the outermost interior ring (C13)."""
    r = np.random.default_rng(seed).standard_normal(shape)
    r[:ring, :] = r[-ring:, :] = 0.0
    r[:, :ring] = r[:, -ring:] = 0.0
    return r


# ----------------------------------------------------------------------------- stencil


def test_laplacian_polynomial_exactness():
    """O3: the 8th-order central 2nd derivative is exact for polynomials of degree <= 9
    (away from the zero-extension boundary). Five even-degree conditions fix the five weights,
    so any wrong weight fails."""
    h = 0.5
    n = 40
    x = (np.arange(n) - n / 2) * h
    for p in range(10):
        u = np.tile(x ** p, (n, 1))                      # varies along J only
        L = wave.laplacian(u, h)[:, 4:-4]
        exact = p * (p - 1) * x[4:-4] ** (p - 2) if p >= 2 else np.zeros(n - 8)
        np.testing.assert_allclose(L[4:-4], np.tile(exact, (n - 8, 1)), rtol=1e-9, atol=1e-6 * max(1, np.abs(exact).max()))
        Lz = wave.laplacian(u.T.copy(), h)[4:-4, :]     # varies along I only
        np.testing.assert_allclose(Lz[:, 4:-4], np.tile(exact, (n - 8, 1)).T, rtol=1e-9,
                                   atol=1e-6 * max(1, np.abs(exact).max()))
    # 2-D mixed monomial: lap(x^3 z^2) = 6 x z^2 + 2 x^3
    Z, X = np.meshgrid(x, x, indexing="ij")
    L = wave.laplacian(X ** 3 * Z ** 2, h)[4:-4, 4:-4]
    ex = (6 * X * Z ** 2 + 2 * X ** 3)[4:-4, 4:-4]
    np.testing.assert_allclose(L, ex, rtol=1e-9, atol=1e-8 * np.abs(ex).max())


def test_laplacian_symmetric_zero_extension():
    """C5: u = 0 outside the padded grid, so <a, L b> = <L a, b> (needed for the exact adjoint)."""
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((2, 17, 23))
    lhs = np.sum(a * wave.laplacian(b, 3.0))
    rhs = np.sum(wave.laplacian(a, 3.0) * b)
    assert abs(lhs - rhs) <= 1e-13 * abs(lhs)


def test_sponge_zero_inside_positive_outside():
    c = wave.sponge_c(10, 14, 5, 10.0, 1e-3, 2000.0)
    assert np.all(c[5:15, 5:19] == 0.0)
    ring = c.copy()
    ring[5:15, 5:19] = 1.0
    assert np.all(ring > 0.0) and c.max() < 1.0


def test_wavelet_ricker_closed_form():
    """O4 / C9: Ricker peak 1 at t0 = 1/f, zero crossings at t0 +- 1/(pi f sqrt 2)."""
    f, dt = 10.0, 1e-4
    s = wlmod.ricker(3000, dt, f).astype(np.float64)
    t = np.arange(3000) * dt
    assert abs(t[np.argmax(s)] - 0.1) < 1.5 * dt and abs(s.max() - 1.0) < 1e-6
    tz = 0.1 + 1.0 / (math.pi * f * math.sqrt(2.0))
    i = int(round(tz / dt))
    assert s[i - 1] * s[i + 1] < 0.0


# ----------------------------------------------------------------------------- P1 / P2


@pytest.mark.parametrize("case", ["tiny", "cfg0"])
def test_adjoint_identity(case):
    """P1: <J dv, rho> = <dv, J^T rho> to <= 1e-10 relative (BASELINE.json north_star)."""
    wl = tiny() if case == "tiny" else wlmod.config(0)
    pb = wave.Problem(wl)
    rng = np.random.default_rng(11)
    dv = rng.standard_normal((wl.nz, wl.nx))
    rho = rng.standard_normal((wl.nt, wl.nrec))
    for shot in range(wl.ns):
        Jdv = pb.born(shot, [dv])[0]
        _, hist = pb.history(shot, "full")
        JTrho = pb.adjoint_image(rho, hist)
        lhs = float(np.sum(Jdv[1:] * rho[1:]))       # rho[0] unused: u^0 is not an unknown
        rhs = float(np.sum(dv * JTrho))
        assert abs(lhs - rhs) <= 1e-10 * max(abs(lhs), abs(rhs)), (lhs, rhs)
        assert np.all(Jdv[0] == 0.0)


def test_hessian_symmetric_psd():
    """P2: H self-adjoint and a normal operator F*F:
    <w, H v> = <v, H w>, <v, H v> = ||J v||^2 >= 0."""
    wl = tiny()
    pb = wave.Problem(wl)
    rng = np.random.default_rng(5)
    v, w = rng.standard_normal((2, wl.nz, wl.nx))
    Hv, Hw = pb.hessvec([v, w])
    a, b = float(np.sum(w * Hv)), float(np.sum(v * Hw))
    assert abs(a - b) <= 1e-10 * max(abs(a), abs(b))
    Jv = np.stack([pb.born(s, [v])[0] for s in range(wl.ns)])
    nrm = float(np.sum(Jv ** 2))
    vHv = float(np.sum(v * Hv))
    assert vHv > 0 and abs(vHv - nrm) <= 1e-12 * nrm


# ----------------------------------------------------------------------------- P3


def test_born_matches_finite_difference():
    """P3(i): [F(v + e dv) - F(v - e dv)] / 2e -> J dv with an O(e^2) error."""
    wl = tiny()
    pb = wave.Problem(wl)
    dv = 30.0 * edge_free((wl.nz, wl.nx), 1)
    Jdv = pb.born(0, [dv])[0]
    errs = []
    for eps in (1e-1, 1e-2):
        fp = wave.Problem(wl, wl.model.astype(np.float64) + eps * dv).forward(0)
        fm = wave.Problem(wl, wl.model.astype(np.float64) - eps * dv).forward(0)
        errs.append(rel_l2((fp - fm) / (2 * eps), Jdv))
    assert errs[1] < 1e-5
    assert errs[1] < errs[0] / 50.0, errs           # ~100x per decade => second order


def test_gradient_fd():
    """P3(ii): [phi(v + e dv) - phi(v - e dv)] / 2e = <g, dv> to <= 1e-6 relative."""
    wl = tiny()
    pt = wave.Problem(wl, wl.model_true)
    d_obs = pt.forward_all()
    pb = wave.Problem(wl)
    phi, g = pb.gradient(d_obs)
    dv = 20.0 * edge_free((wl.nz, wl.nx), 2)
    eps = 1e-4

    def phi_at(m):
        p = wave.Problem(wl, m)
        r = p.forward_all() - d_obs
        return 0.5 * float(np.sum(r * r))
    m = wl.model.astype(np.float64)
    fd = (phi_at(m + eps * dv) - phi_at(m - eps * dv)) / (2 * eps)
    an = float(np.sum(g * dv))
    assert phi > 0
    assert abs(fd - an) <= 1e-6 * abs(an), (fd, an)


def test_hessian_is_gradient_derivative_at_zero_residual():
    """P3(iii): at zero residual GN = full Hessian, so [g(v + e w) - g(v - e w)] / 2e -> H w, O(e^2)."""
    wl = tiny()
    pb = wave.Problem(wl)
    d_obs = pb.forward_all()
    w = 20.0 * edge_free((wl.nz, wl.nx), 4)
    Hw = pb.hessvec([w])[0]
    m = wl.model.astype(np.float64)
    errs = []
    for eps in (1e-1, 1e-2):
        gp = wave.Problem(wl, m + eps * w).gradient(d_obs)[1]
        gm = wave.Problem(wl, m - eps * w).gradient(d_obs)[1]
        errs.append(rel_l2((gp - gm) / (2 * eps), Hw))
    assert errs[1] < 1e-5 and errs[1] < errs[0] / 50.0, errs


# ----------------------------------------------------------------------------- P4


def _green_trace(r, c, t, wavelet_fn, nsig=4000):
    """u(r, t) = int_{r/c}^{t} G(r, tau) s(t - tau) dtau, G = H(c tau - r) / (2 pi c sqrt(c^2 tau^2 - r^2)),
    with tau = r/c + sigma^2 to remove the square-root singularity."""
    out = np.zeros_like(t)
    for i, ti in enumerate(t):
        if ti <= r / c:
            continue
        smax = math.sqrt(ti - r / c)
        sig = np.linspace(0.0, smax, nsig)
        tau = r / c + sig ** 2
        integrand = wavelet_fn(ti - tau) / (math.pi * c * np.sqrt(c) * np.sqrt(c * tau + r))
        out[i] = np.trapezoid(integrand, sig)
    return out


def test_homogeneous_green_function_and_traveltime():
    """P4: homogeneous v = 2000 m/s, 96x96, h = 10 m, dt = 1 ms, 10 Hz Ricker, centred source.
    The traces match the closed-form 2-D Green's function convolved with s (2-D wave equation
    u_tt = c^2 lap u + s(t) delta(x)), and cross-correlation lags equal offset / c."""
    c, h, dt, f, nt = 2000.0, 10.0, 1e-3, 10.0, 400
    wl = wlmod.custom(96, 96, h=h, dt=dt, nt=nt, W=20, ns=1, f_peak=f, model_kind="homogeneous",
                      v_ref=c)
    wl.src = np.array([[48, 48]], dtype=np.int32)
    offs = np.array([10, 15, 20, 25, 30])
    wl.rec = np.stack([np.full(len(offs), 48), 48 + offs], axis=1).astype(np.int32)
    d = wave.Problem(wl).forward(0)
    t = np.arange(nt) * dt
    t0 = 1.0 / f

    def s_fn(tt):
        a = (math.pi * f * (tt - t0)) ** 2
        return np.where(tt >= 0, (1 - 2 * a) * np.exp(-a), 0.0)
    for i, o in enumerate(offs):
        r = o * h
        g = _green_trace(r, c, t, s_fn)
        win = t < (r / c + t0 + 0.1)           # before any sponge reflection returns
        assert rel_l2(d[win, i], g[win]) < 0.03, (o, rel_l2(d[win, i], g[win]))
    # travel-time differences from cross-correlation, sub-sample by parabolic fit
    ref = d[:, 0]
    for i, o in enumerate(offs[1:], start=1):
        xc = np.correlate(d[:, i], ref, mode="full")
        k = int(np.argmax(xc))
        y0, y1, y2 = xc[k - 1], xc[k], xc[k + 1]
        frac = 0.5 * (y0 - y2) / (y0 - 2 * y1 + y2)
        lag = (k - (nt - 1) + frac) * dt
        expect = (o - offs[0]) * h / c
        assert abs(lag - expect) <= max(2 * dt, 0.01 * expect), (o, lag, expect)


# ----------------------------------------------------------------------------- P5


def test_reciprocity():
    """P5: v(x_s)^2 d_{s->r}(t) = v(x_r)^2 d_{r->s}(t) in a heterogeneous model with sponge
    (the M-scaled scheme has spatially symmetric blocks). Without the v^2 weights it fails."""
    wl = tiny(nz=14, nx=18, nt=90)
    a, b = (3, 4), (9, 13)
    m = wl.model.astype(np.float64)
    wl1 = wl.subset()
    wl1.src = np.array([a], dtype=np.int32)
    wl1.rec = np.array([b], dtype=np.int32)
    wl2 = wl.subset()
    wl2.src = np.array([b], dtype=np.int32)
    wl2.rec = np.array([a], dtype=np.int32)
    dab = wave.Problem(wl1).forward(0)[:, 0]
    dba = wave.Problem(wl2).forward(0)[:, 0]
    lhs = m[a] ** 2 * dab
    rhs = m[b] ** 2 * dba
    assert rel_l2(lhs, rhs) <= 1e-12
    assert rel_l2(dab, dba) > 1e-3                    # the weights matter (v differs at a, b)


# ----------------------------------------------------------------------------- P6


def test_brute_force_dense_J():
    """P6: build J densely from Born runs on all unit vectors (12x12 interior, W = 6, nt = 80);
    J^T equals the dense transpose, H = J^T J is symmetric PSD and equals the oracle's H v."""
    wl = tiny()
    pb = wave.Problem(wl)
    N = wl.nz * wl.nx
    E = np.eye(N).reshape(N, wl.nz, wl.nx)
    rng = np.random.default_rng(9)
    H = np.zeros((N, N))
    for s in range(wl.ns):
        Jd = pb.born(s, list(E))                             # [N][nt][nrec]
        J = Jd.reshape(N, -1).T                              # [(nt nrec)][N]
        rho = rng.standard_normal((wl.nt, wl.nrec))
        _, hist = pb.history(s, "full")
        JT = pb.adjoint_image(rho, hist).ravel()
        ref = J.T @ rho.ravel()
        assert rel_l2(JT, ref) <= 1e-12
        H += J.T @ J
    assert np.max(np.abs(H - H.T)) <= 1e-12 * np.max(np.abs(H))
    ev = np.linalg.eigvalsh(0.5 * (H + H.T))
    assert ev.min() >= -1e-12 * ev.max()
    v = rng.standard_normal((wl.nz, wl.nx))
    assert rel_l2(pb.hessvec([v])[0].ravel(), H @ v.ravel()) <= 1e-12


# ----------------------------------------------------------------------------- P7 / P8 / P9


def test_linearity_batching_sharding():
    """P7: H(a v + b w) = a Hv + b Hw; batched = single calls (bitwise); sum over source shards
    = all-source result; H 0 = 0."""
    wl = tiny(ns=3)
    pb = wave.Problem(wl)
    rng = np.random.default_rng(1)
    v, w = rng.standard_normal((2, wl.nz, wl.nx))
    Hv, Hw, Hc = pb.hessvec([v, w, 2.0 * v - 3.0 * w])
    assert rel_l2(Hc, 2.0 * Hv - 3.0 * Hw) <= 1e-12
    Hv1 = pb.hessvec([v])[0]
    assert np.array_equal(Hv1, Hv)
    part = pb.hessvec([v], shots=[0]) + pb.hessvec([v], shots=[1, 2])
    assert rel_l2(part[0], Hv) <= 1e-12
    assert np.all(pb.hessvec([np.zeros_like(v)])[0] == 0.0)


def test_storage_mode_invariance():
    """P8: FULL, CHECKPOINT-replay and BOUNDARY-ring reconstruction give the same H v and g."""
    wl = tiny(nt=97)
    pb = wave.Problem(wl)
    v = np.random.default_rng(2).standard_normal((wl.nz, wl.nx))
    ref = pb.hessvec([v], mode="full")[0]
    for mode, k in (("checkpoint", 7), ("checkpoint", 10), ("checkpoint", 96), ("boundary", 0)):
        out = pb.hessvec([v], mode=mode, ckpt=k)[0]
        assert rel_l2(out, ref) <= 1e-12, (mode, k, rel_l2(out, ref))
    d_obs = wave.Problem(wl, wl.model_true).forward_all()
    _, g0 = pb.gradient(d_obs, mode="full")
    _, g1 = pb.gradient(d_obs, mode="checkpoint", ckpt=9)
    _, g2 = pb.gradient(d_obs, mode="boundary")
    assert rel_l2(g1, g0) <= 1e-12 and rel_l2(g2, g0) <= 1e-12


def test_translation_invariance():
    """P9: homogeneous medium, source and receivers shifted by whole cells, before the wave
    reaches the sponge -> identical traces (stencil symmetry and indexing)."""
    wl = wlmod.custom(60, 60, nt=60, W=10, ns=1, f_peak=30.0, model_kind="homogeneous", v_ref=2000.0)
    wl.src = np.array([[20, 22]], dtype=np.int32)
    wl.rec = np.array([[20, 30], [26, 22], [14, 17]], dtype=np.int32)
    d1 = wave.Problem(wl).forward(0)
    wl2 = wl.subset()
    wl2.src = wl.src + np.array([[7, 9]], dtype=np.int32)
    wl2.rec = wl.rec + np.array([[7, 9]], dtype=np.int32)
    d2 = wave.Problem(wl2).forward(0)
    assert np.linalg.norm(d1) > 0
    assert rel_l2(d2, d1) <= 1e-12
    # mirror symmetry of the stencil: receivers mirrored about the source see the same trace
    wl3 = wl.subset()
    wl3.rec = np.array([[20, 14], [14, 22], [26, 27]], dtype=np.int32)
    d3 = wave.Problem(wl3).forward(0)
    assert rel_l2(d3, d1) <= 1e-12


def test_sponge_absorbs():
    """C4 / C10: the centred sponge absorbs: 1 s after a 15 Hz pulse in a 600 m box, the traces
    are < 0.5 % of their peak (mis-centred damping or a too-weak profile leaves 9-28 %)."""
    wl = wlmod.custom(60, 60, nt=1200, W=20, ns=1, f_peak=15.0, model_kind="homogeneous", v_ref=2000.0)
    wl.src = np.array([[30, 30]], dtype=np.int32)
    wl.rec = np.array([[30, 30], [10, 10], [50, 45]], dtype=np.int32)
    d = wave.Problem(wl).forward(0)
    assert np.abs(d[-200:]).max() < 5e-3 * np.abs(d).max()
