"""GPU parity: the CUDA path through the C ABI vs the fp64 oracle on the same seeded inputs (P10).

Bar (BASELINE.json north_star): relative L2 <= 1e-4 on d, g and H·v. Cases span several 64x32 tiles
with ragged tails, every storage mode, several shot batches and field groupings, and full BASELINE
sizes (properties that hold at any size here; the bench's exact launch plans against oracle golden rows
in tests/test_gpu_golden.py)."""
import numpy as np
import pytest

from oracle import psido as opsido
from oracle import wave
from tests.conftest import rel_l2
import workloads as W

pytestmark = pytest.mark.gpu

TOL = 1e-4
PHI_TOL = 2 * TOL   # phi = 1/2 |rho|^2 is quadratic in rho: rel(phi) ~ 2 rel_l2(rho)


@pytest.fixture(scope="module")
def hv():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2507_10804_b200 as hvmod
    return hvmod


# ---------------------------------------------------------------------------------------------- cfg 0


@pytest.fixture(scope="module")
def cfg0_ref():
    wl = W.config(0)
    pb = wave.Problem(wl)
    V = wl.probes()
    d = pb.forward_all()
    HV = pb.hessvec(list(V.astype(np.float64)))
    # gradient recipe (DESIGN.md §3 R-grad): d_obs = F(model) from the oracle (fp32-rounded, C17), evaluated at
    # a 4 % slow starting model, so the residual is O(|d|) and fp32 rounding of d is not amplified
    m0 = (0.96 * W.m0_cfg0()).astype(np.float32)
    d_obs = d.astype(np.float32)
    phi, g = wave.Problem(wl, m0).gradient(d_obs)
    return wl, V, d, HV, m0, d_obs, phi, g


def test_cfg0_forward(hv, cfg0_ref):
    wl, V, d, *_ = cfg0_ref
    s = hv.Solver.from_workload(wl)
    dg = s.forward(wl.model)
    assert dg.shape == d.shape
    assert np.all(dg[:, 0, :] == 0.0)
    assert rel_l2(dg, d) <= TOL, rel_l2(dg, d)


@pytest.mark.parametrize("store", ["full", "checkpoint", "boundary"])
def test_cfg0_hessvec(hv, cfg0_ref, store):
    wl, V, d, HV, *_ = cfg0_ref
    s = hv.Solver.from_workload(wl, store=store)
    out = s.hessvec(wl.model, V)
    assert rel_l2(out, HV) <= TOL, rel_l2(out, HV)
    assert s.stats()["store"] == hv.STORE[store]


def test_cfg0_gradient(hv, cfg0_ref):
    wl, V, d, HV, m0, d_obs, phi, g = cfg0_ref
    s = hv.Solver.from_workload(wl)
    phig, gg = s.gradient(m0, d_obs)
    assert rel_l2(gg, g) <= TOL, rel_l2(gg, g)
    assert abs(phig - phi) <= PHI_TOL * phi


def test_cfg0_gradient_near_zero_residual(hv, cfg0_ref):
    """The SURVEY.md §8(d) recipe (m0 = anomaly removed) leaves a residual of only 0.28 % of |d|, so the fp32
    rounding of the forward data (eps_d <= 1e-5 relative) is amplified by |d| / |rho| in
    rho = d - d_obs. Derived bound: rel_l2(g) <= 1e-4 + 2 eps_d |d| / |rho|."""
    wl, V, d, HV, m0, d_obs, phi, g = cfg0_ref
    m1 = W.m0_cfg0()
    pb = wave.Problem(wl, m1)
    phi1, g1 = pb.gradient(d_obs)
    rho = pb.forward_all() - d_obs
    ratio = np.linalg.norm(d_obs) / np.linalg.norm(rho)
    s = hv.Solver.from_workload(wl)
    phig, gg = s.gradient(m1, d_obs)
    tol = 1e-4 + 2 * 1e-5 * ratio
    assert rel_l2(gg, g1) <= tol, (rel_l2(gg, g1), tol)
    assert abs(phig - phi1) <= tol * phi1


def test_cfg0_fused_gradient_hessvec(hv, cfg0_ref):
    wl, V, d, HV, m0, d_obs, phi, g = cfg0_ref
    s = hv.Solver.from_workload(wl)
    pb = wave.Problem(wl, m0)
    HV0 = pb.hessvec(list(V.astype(np.float64)))
    phig, gg, hvg = s.gradient_hessvec(m0, d_obs, V)
    assert rel_l2(gg, g) <= TOL and rel_l2(hvg, HV0) <= TOL
    assert abs(phig - phi) <= PHI_TOL * phi


# ---------------------------------------------------------------------------------------------- multi-tile


@pytest.fixture(scope="module")
def ragged():
    """70 x 150 interior (110 x 190 padded: 4 x 3 tiles of 32 x 64, ragged in both directions),
    3 shots, 3 probes, sparse receiver line, nt = 300."""
    wl = W.custom(70, 150, nt=300, ns=3, nrec=37, n_probes=3, f_peak=15.0, seed=5)
    pb = wave.Problem(wl)
    V = wl.probes()
    d = pb.forward_all()
    HV = pb.hessvec(list(V.astype(np.float64)))
    d_obs = wave.Problem(wl, wl.model_true).forward_all().astype(np.float32)
    m_start = (0.96 * wl.model).astype(np.float32)          # well-conditioned residual (R-grad)
    phi, g = wave.Problem(wl, m_start).gradient(d_obs)
    return wl, V, d, HV, d_obs, phi, g, m_start


@pytest.mark.parametrize("store,ckpt,batch,fg", [
    ("full", 0, 1, 8), ("full", 0, 2, 1), ("full", 0, 3, 2),
    ("checkpoint", 7, 1, 8), ("checkpoint", 0, 3, 1), ("checkpoint", 299, 2, 3),
    ("boundary", 0, 1, 8), ("boundary", 0, 3, 2),
])
def test_ragged_hessvec_modes(hv, ragged, store, ckpt, batch, fg):
    wl, V, d, HV, *_ = ragged
    s = hv.Solver.from_workload(wl, store=store, ckpt_interval=ckpt, shot_batch=batch, field_group=fg)
    out = s.hessvec(wl.model, V)
    assert rel_l2(out, HV) <= TOL, rel_l2(out, HV)
    for k in range(3):
        assert rel_l2(out[k], HV[k]) <= TOL


@pytest.mark.parametrize("store", ["full", "checkpoint", "boundary"])
def test_ragged_forward_gradient(hv, ragged, store):
    wl, V, d, HV, d_obs, phi, g, m_start = ragged
    s = hv.Solver.from_workload(wl, shot_batch=2, store=store)
    assert rel_l2(s.forward(wl.model), d) <= TOL
    phig, gg = s.gradient(m_start, d_obs)
    assert rel_l2(gg, g) <= TOL and abs(phig - phi) <= PHI_TOL * phi


def test_ragged_shards_sum(hv, ragged):
    """Source sharding (a8): partial sums over [0,1) + [1,3) equal the full result (rank-local sums)."""
    wl, V, d, HV, *_ = ragged
    a = hv.Solver.from_workload(wl, src_begin=0, src_end=1).hessvec(wl.model, V)
    b = hv.Solver.from_workload(wl, src_begin=1, src_end=3).hessvec(wl.model, V)
    assert rel_l2(a + b, HV) <= TOL
    ref1 = wave.Problem(wl).hessvec(list(V.astype(np.float64)), shots=[0])
    assert rel_l2(a, ref1) <= TOL


def test_device_pointers_match_host_pointers(hv, ragged):
    import torch
    wl, V, d, HV, *_ = ragged
    s = hv.Solver.from_workload(wl)
    host = s.hessvec(wl.model, V)
    dev = s.hessvec(torch.from_numpy(wl.model).cuda(), torch.from_numpy(V).cuda())
    assert isinstance(dev, torch.Tensor) and dev.is_cuda
    assert np.array_equal(dev.cpu().numpy(), host)           # bitwise: same kernels, same order


def test_deterministic_and_batch_invariant(hv, ragged):
    wl, V, *_ = ragged
    s = hv.Solver.from_workload(wl, shot_batch=1, field_group=1)
    a = s.hessvec(wl.model, V)
    b = s.hessvec(wl.model, V)
    assert np.array_equal(a, b)
    # probe k alone equals row k of the batch (each field's arithmetic is independent of the grouping)
    c = s.hessvec(wl.model, V[1:2])
    assert np.array_equal(c[0], a[1])


@pytest.mark.parametrize("nt,K", [(300, 3), (301, 7), (161, 9)])
def test_t2_kernels_match_single_step(hv, nt, K, monkeypatch):
    """The T = 2 forward (fwd_t2_kernel: two levels per launch, resident q_k, groups of <= 4 Born fields) and
    adjoint (bwd_t2_kernel) compute every level with the single-step kernels' per-point operations: d, g, phi and
    H·v agree with HV_T2=0 to rounding. Even and odd numbers of steps (nt - 1: a trailing one-level launch), one
    and several Born-field groups; and against the oracle."""
    wl = W.custom(70, 150, nt=nt, ns=3, nrec=37, n_probes=K, f_peak=15.0, seed=5)
    V = wl.probes()
    d_obs = np.zeros((wl.ns, wl.nt, wl.nrec), np.float32)
    out = {}
    for t2, t2b in (("1", "0"), ("0", "0"), ("1", "1")):
        monkeypatch.setenv("HV_T2", t2)
        monkeypatch.setenv("HV_T2B", t2b)
        s = hv.Solver.from_workload(wl, store="full", shot_batch=2)
        out[t2 + t2b] = (s.forward(wl.model), s.gradient(wl.model, d_obs), s.hessvec(wl.model, V))
        assert s.stats()["fwd_kernel"] == (3 if t2 == "1" else 0)
        assert s.stats()["bwd_kernel"] == (3 if t2b == "1" else 0)
    (d1, (p1, g1), h1), (d0, (p0, g0), h0) = out["10"], out["00"]
    # same per-point operations; since the background runs in increment form the T = 2 and single-step paths
    # differ by isolated 1-ulp roundings at the wavefront (measured 6e-8 relative), so: rounding-level agreement
    assert rel_l2(d1, d0) <= 1e-6 and abs(p1 - p0) <= 1e-6 * p0
    assert rel_l2(g1, g0) <= 1e-6 and rel_l2(h1, h0) <= 1e-6
    # T = 2 adjoint: imaging summed two levels per launch (fp32 summation order)
    d2, (p2, g2), h2 = out["11"]
    assert np.array_equal(d2, d1) and p2 == p1
    assert rel_l2(g2, g0) <= 1e-6 and rel_l2(h2, h0) <= 1e-6
    ref = wave.Problem(wl).hessvec(list(V.astype(np.float64)))
    assert rel_l2(h1, ref) <= TOL and rel_l2(h2, ref) <= TOL


@pytest.mark.parametrize("nz,nx,ns,K,fg,batch", [
    (5, 200, 3, 7, 3, 1),      # a one-tile-row grid, 7 Born fields in near-equal groups of <= 3, 1 shot per batch
    (150, 7, 2, 17, 0, 0),     # a one-tile-column grid, auto field groups (busiest-CTA model) for K = 17
    (40, 300, 5, 1, 0, 2),     # K = 1, 5 shots in batches of 2 (ragged last batch)
])
def test_schedule_shapes(hv, nz, nx, ns, K, fg, batch):
    """Forward one-wave schedule and backward grid on degenerate shapes: thin grids, K not a multiple of the group
    size, a single probe, ragged shot batches -- H·v against the oracle."""
    wl = W.custom(nz, nx, nt=120, ns=ns, nrec=max(2, nx // 3), n_probes=K, f_peak=20.0, seed=3)
    V = wl.probes()
    ref = wave.Problem(wl).hessvec(list(V.astype(np.float64)))
    out = hv.Solver.from_workload(wl, shot_batch=batch, field_group=fg).hessvec(wl.model, V)
    assert rel_l2(out, ref) <= TOL
    for k in range(K):
        assert rel_l2(out[k], ref[k]) <= TOL


def test_unit_order_shot_blocks_bitwise(hv, monkeypatch):
    """The forward unit order (shot blocks of HV_SBLK shots, a ragged last block) only reorders independent
    items: d and H·v are bitwise equal for every block size."""
    wl = W.custom(70, 150, nt=160, ns=5, nrec=30, n_probes=5, f_peak=15.0, seed=9)
    V = wl.probes()
    res = []
    for b in ("1", "3", "5"):
        monkeypatch.setenv("HV_SBLK", b)
        s = hv.Solver.from_workload(wl, shot_batch=5, field_group=2)
        res.append((s.forward(wl.model), s.hessvec(wl.model, V)))
    for d, h in res[1:]:
        assert np.array_equal(d, res[0][0]) and np.array_equal(h, res[0][1])


@pytest.mark.parametrize("store", ["full", "checkpoint", "boundary"])
def test_resident_q_forward(hv, ragged, store, monkeypatch):
    """The resident-q forward (chosen for Q larger than L2; forced here with HV_QRES=1) against the oracle and
    against the one-wave forward."""
    wl, V, d, HV, *_ = ragged
    out = {}
    for q in ("1", "0"):
        monkeypatch.setenv("HV_QRES", q)
        monkeypatch.setenv("HV_QFG", "2")
        s = hv.Solver.from_workload(wl, store=store, shot_batch=2)
        out[q] = (s.forward(wl.model), s.hessvec(wl.model, V))
    assert rel_l2(out["1"][0], d) <= TOL and rel_l2(out["1"][1], HV) <= TOL
    assert rel_l2(out["1"][0], out["0"][0]) <= 1e-6 and rel_l2(out["1"][1], out["0"][1]) <= 1e-6
    # thread-block-cluster variant (experimental, off by default): background once per tile, shared by DSMEM
    monkeypatch.setenv("HV_QRES", "1")
    monkeypatch.setenv("HV_QRES_CLUSTER", "1")
    s = hv.Solver.from_workload(wl, store=store, shot_batch=2)
    hcl = s.hessvec(wl.model, V)
    assert s.stats()["fwd_kernel"] == 4
    assert rel_l2(hcl, HV) <= TOL and rel_l2(hcl, out["1"][1]) <= 1e-6


def test_edge_cases(hv):
    # degenerate: zero probe -> zero H v, zero residual -> zero gradient; minimum grid; receiver on a corner
    wl = W.custom(1, 5, nt=40, ns=1, nrec=2, n_probes=1, W=4, f_peak=25.0, seed=2)
    wl.rec = np.array([[0, 0], [0, 4]], dtype=np.int32)
    wl.src = np.array([[0, 2]], dtype=np.int32)
    s = hv.Solver.from_workload(wl)
    z = s.hessvec(wl.model, np.zeros((1, 1, 5), np.float32))
    assert np.all(z == 0.0)
    ref = wave.Problem(wl)
    d = s.forward(wl.model)
    assert rel_l2(d, ref.forward_all()) <= TOL
    phi, g = s.gradient(wl.model, d)
    assert phi == 0.0 and np.all(g == 0.0)
    V = wl.probes()
    assert rel_l2(s.hessvec(wl.model, V), ref.hessvec(list(V.astype(np.float64)))) <= TOL


def test_forward_only_t2_default(hv, monkeypatch):
    """Forward-only calls on a grid with at least one T = 2 tile per SM (the cfg 3 grid) run the T = 2 forward by
    default; d and the misfit agree with the single-step kernels (HV_T2=0) to rounding (the increment-form
    background makes isolated 1-ulp differences, as in test_t2_kernels_match_single_step) and with the gradient's
    phi (single-step forward)."""
    wl = W.config(3).subset(shots=range(3), nt=300)
    monkeypatch.delenv("HV_T2", raising=False)
    s = hv.Solver.from_workload(wl)
    d = s.forward(wl.model)
    assert s.stats()["fwd_kernel"] == 3
    m0 = (0.98 * wl.model).astype(np.float32)
    phi = s.misfit(m0, d)
    assert s.stats()["fwd_kernel"] == 3
    phig, _ = s.gradient(m0, d)
    assert phi > 0 and abs(phi - phig) <= 1e-6 * phig
    monkeypatch.setenv("HV_T2", "0")
    s0 = hv.Solver.from_workload(wl)
    d0 = s0.forward(wl.model)
    assert s0.stats()["fwd_kernel"] != 3
    assert rel_l2(d, d0) <= 1e-6
    assert abs(s0.misfit(m0, d) - phi) <= 1e-6 * phi


def test_duplicate_receivers(hv):
    """Two receivers on one node (and one on a tile corner): the adjoint's R^T injects both (receiver chain of the
    backward kernel's per-tile map) and the gradient and H·v match the oracle."""
    wl = W.custom(40, 70, nt=120, ns=2, nrec=5, n_probes=2, W=6, f_peak=20.0, seed=5)
    wl.rec = np.array([[2, 10], [2, 10], [2, 31], [9, 63], [2, 10]], dtype=np.int32)
    ref = wave.Problem(wl)
    s = hv.Solver.from_workload(wl)
    V = wl.probes()
    assert rel_l2(s.hessvec(wl.model, V), ref.hessvec(list(V.astype(np.float64)))) <= TOL
    d_obs = wave.Problem(wl, wl.model_true).forward_all().astype(np.float32)
    m0 = (0.96 * wl.model).astype(np.float32)
    phi, g = s.gradient(m0, d_obs)
    phi_ref, g_ref = wave.Problem(wl, m0).gradient(d_obs)
    assert abs(phi - phi_ref) <= 2 * TOL * phi_ref and rel_l2(g, g_ref) <= TOL


def test_errors(hv):
    wl = W.config(0)
    s = hv.Solver.from_workload(wl)
    with pytest.raises(hv.HVError) as e:
        s.forward(wl.model * 100.0)          # violates CFL
    assert e.value.status == hv.HV_ECFL
    bad = W.config(0)
    bad.src = np.array([[64, 0]], dtype=np.int32)
    with pytest.raises(hv.HVError) as e:
        hv.Solver.from_workload(bad)
    assert e.value.status == hv.HV_EINVAL


# ---------------------------------------------------------------------------------------------- full size


def test_cfg1_full_batch_properties(hv):
    """All 16 shots x 64 PSF spikes (the bench workload): H symmetric on the spike lattice,
    HV_i(x_j) = HV_j(x_i) (self-adjoint), PSD diagonal, and batching invariance."""
    wl = W.config(1)
    V = wl.probes()
    s = hv.Solver.from_workload(wl, shot_batch=2)
    out = s.hessvec(wl.model, V).astype(np.float64)
    pts = [tuple(np.argwhere(v)[0]) for v in V]
    M = np.array([[out[i][pts[j]] for j in range(64)] for i in range(64)])
    scale = np.abs(np.diag(M)).max()
    assert np.all(np.diag(M) > 0)
    assert np.max(np.abs(M - M.T)) <= 1e-4 * scale
    # storage-mode invariance at full size (P8 on the GPU): BOUNDARY reverses 2000 fp32 leapfrog steps
    for store in ("checkpoint", "boundary"):
        alt = hv.Solver.from_workload(wl, shot_batch=2, store=store).hessvec(wl.model, V)
        assert rel_l2(alt, out) <= TOL, (store, rel_l2(alt, out))
    sub = s.hessvec(wl.model, V[[5, 40]])            # same shot batching -> bitwise identical rows
    assert np.array_equal(sub[0], out[5].astype(np.float32)) and np.array_equal(sub[1], out[40].astype(np.float32))


# ---------------------------------------------------------------------------------------------- PsiDO


@pytest.mark.parametrize("nz,nx,r", [(16, 24, 1), (33, 47, 3), (64, 128, 8)])
def test_psido_apply_parity(hv, nz, nx, r):
    rng = np.random.default_rng(nz * nx + r)
    a = rng.standard_normal((r, nz, nx)).astype(np.float32)
    b = (rng.standard_normal((r, nz, nx)) + 1j * rng.standard_normal((r, nz, nx))).astype(np.complex64)
    v = rng.standard_normal((nz, nx)).astype(np.float32)
    s = hv.Solver.from_workload(W.config(0))
    for mode in range(3):
        out = s.psido_apply(a, b, v, mode)
        ref = opsido.apply_mode(a.astype(np.float64), b.astype(np.complex128), v.astype(np.float64), mode)
        assert rel_l2(out, ref) <= TOL, (mode, rel_l2(out, ref))


# ---------------------------------------------------------------------------------------------- cfg 4
# Full-nt oracle comparisons of the cfg 1 / 2 / 3 bench plans use committed golden rows (tests/test_gpu_golden.py).
# The cfg 4 grid (2048 x 6144, 12.9 M padded points) is checked on a truncated time axis: the fp64 numpy oracle
# needs ~0.5 s per field-step there.


def test_cfg4_full_grid_checkpoint_slice(hv):
    """2048 x 6144 (12.9 M padded points) in CHECKPOINT mode: shot 127, probe 0, nt truncated to 48 (the fp64 numpy
    oracle needs ~0.5 s per field-step on this grid)."""
    wl = W.config(4).subset(shots=[127], nt=48)
    V = wl.probes([0])
    ref = wave.Problem(wl).hessvec(list(V.astype(np.float64)), mode="checkpoint", ckpt=7)
    s = hv.Solver.from_workload(wl, store="checkpoint", ckpt_interval=5)
    out = s.hessvec(wl.model, V)
    assert s.stats()["store"] == 2
    assert rel_l2(out, ref) <= TOL, rel_l2(out, ref)
