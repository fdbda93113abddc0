"""C-ABI calls beyond the H·v itself: per-shot forward, misfit-only (gpCN) call, empty shards,
in-library NCCL reduction, stream ordering against torch's default stream, model validation."""
import numpy as np
import pytest

from oracle import wave
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
def case():
    return W.custom(70, 150, nt=300, ns=3, nrec=37, n_probes=3, f_peak=15.0, seed=5)


def test_forward_shot(hv, case):
    """hv_forward_shot(isrc) equals row isrc - src_begin of the shard forward bitwise, and the oracle's f_s(m)
    (PAPER.md:49); a shot outside the shard is HV_EINVAL."""
    s = hv.Solver.from_workload(case, src_begin=1, src_end=3)
    full = s.forward(case.model)
    for isrc in (1, 2):
        d = s.forward_shot(case.model, isrc)
        assert np.array_equal(d, full[isrc - 1])
        assert rel_l2(d, wave.Problem(case).forward(isrc)) <= TOL
    for bad in (0, 3, -1):
        with pytest.raises(hv.HVError) as e:
            s.forward_shot(case.model, bad)
        assert e.value.status == hv.HV_EINVAL


def test_misfit_only(hv, case):
    """hv_misfit (forward + residual, no adjoint; the gpCN likelihood) equals the oracle's
    phi and, bitwise, the phi of hv_gradient (same forward kernels, same fixed-order reduction)."""
    s = hv.Solver.from_workload(case)
    d_obs = wave.Problem(case, case.model_true).forward_all().astype(np.float32)
    m0 = (0.96 * case.model).astype(np.float32)
    phi = s.misfit(m0, d_obs)
    pb = wave.Problem(case, m0)
    res = pb.forward_all() - d_obs
    phi_ref = 0.5 * float(np.sum(res * res))
    assert abs(phi - phi_ref) <= 2 * TOL * phi_ref
    phig, _ = s.gradient(m0, d_obs)
    assert phi == phig
    assert s.misfit(m0, d_obs) == phi                      # deterministic (no atomics)


def test_gradient_phi_bit_deterministic(hv, case):
    s = hv.Solver.from_workload(case, shot_batch=2)
    d_obs = np.zeros((case.ns, case.nt, case.nrec), np.float32)
    a = s.gradient(case.model, d_obs)
    b = s.gradient(case.model, d_obs)
    assert a[0] == b[0] and np.array_equal(a[1], b[1])


def test_empty_shard(hv, case):
    """More ranks than shots leaves a rank with an empty shard: its partial sums are zero."""
    s = hv.Solver.from_workload(case, src_begin=2, src_end=2)
    V = case.probes()
    assert np.all(s.hessvec(case.model, V) == 0.0)
    phi, g = s.gradient(case.model, np.zeros((0, case.nt, case.nrec), np.float32))
    assert phi == 0.0 and np.all(g == 0.0)
    assert s.forward(case.model).shape == (0, case.nt, case.nrec)


def test_in_library_nccl_one_rank(hv, case):
    """The in-library all-reduce path (hv_set_comm) on a 1-rank communicator: result bitwise equal to no comm."""
    uid = hv.nccl_unique_id()
    comm = hv.nccl_comm_create(1, 0, uid, 0)
    try:
        V = case.probes()
        ref = hv.Solver.from_workload(case).hessvec(case.model, V)
        s = hv.Solver.from_workload(case, nccl_comm=comm)
        assert np.array_equal(s.hessvec(case.model, V), ref)
        d_obs = np.zeros((case.ns, case.nt, case.nrec), np.float32)
        s2 = hv.Solver.from_workload(case)
        assert s.gradient(case.model, d_obs)[0] == s2.gradient(case.model, d_obs)[0]
        phi_c = s.misfit(case.model, d_obs)
        assert phi_c == s2.misfit(case.model, d_obs)
        # the eigensolver's batched H·v go through the same in-library reduction
        Om = np.random.default_rng(3).standard_normal((6, case.nz, case.nx)).astype(np.float32)
        ev_c, _ = s.lowrank_geneig(case.model, Om, 3, power_iters=1)
        ev_r, _ = s2.lowrank_geneig(case.model, Om, 3, power_iters=1)
        assert np.array_equal(ev_c, ev_r)
        s.set_comm(None)
        assert np.array_equal(s.hessvec(case.model, V), ref)
        s.close()
    finally:
        hv.nccl_comm_destroy(comm)


def test_torch_default_stream_inputs_are_ordered(hv, case):
    """Inputs produced by torch on its default stream (torch.randn on the device, then an elementwise op) are
    complete before the library reads them (the library's own stream waits for the legacy stream)."""
    import torch
    s = hv.Solver.from_workload(case)
    torch.manual_seed(0)
    for _ in range(3):
        big = torch.randn(64 << 20, device="cuda")          # keep the default stream busy
        V = torch.randn((3, case.nz, case.nx), device="cuda")
        V = V * 2.0 + big[:1].abs() * 0.0                      # still in flight when hessvec is called
        out = s.hessvec(torch.from_numpy(case.model).cuda(), V)
        ref = s.hessvec(case.model, V.cpu().numpy())
        assert np.array_equal(out.cpu().numpy(), ref)


def test_model_must_be_positive(hv, case):
    s = hv.Solver.from_workload(case)
    m = case.model.copy()
    m[10, 20] = 0.0
    with pytest.raises(hv.HVError) as e:
        s.forward(m)
    assert e.value.status == hv.HV_EINVAL
    m[10, 20] = -5.0
    with pytest.raises(hv.HVError) as e:
        s.hessvec(m, case.probes())
    assert e.value.status == hv.HV_EINVAL
