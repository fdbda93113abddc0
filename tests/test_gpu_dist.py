"""Multi-rank H·v through the REAL library: two ranks share cuda:0 under the gloo backend, each
runs a `Solver` on its shard (shots, or probe rows when there are fewer shots than ranks) and `ShardedOperator`
all-reduces the partial sums -- the code path bench.py runs at N > 1. The ranks' kernels never wait on each
other (the reduction is host-side gloo), so one GPU is enough. Compared with the 1-rank H·v of the same inputs."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import workloads as W  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(ns):
    return W.custom(70, 150, nt=200, ns=ns, nrec=37, n_probes=3, f_peak=15.0, seed=5)


def _worker(rank, world, port, outdir, ns):
    import torch
    import torch.distributed as dist

    from paper_2507_10804_b200.dist import solver_operator
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    wl = _case(ns)
    op = solver_operator(wl, rank, world, device=0)
    m = torch.from_numpy(wl.model).cuda()
    V = torch.from_numpy(wl.probes()).cuda()
    HV = op.hessvec(m, V)
    sh = op.shard
    d_obs = torch.zeros((sh.s1 - sh.s0, wl.nt, wl.nrec), dtype=torch.float32, device="cuda")
    phi, g = op.gradient(m, d_obs)
    if rank == 0:
        np.save(os.path.join(outdir, "hv.npy"), HV.cpu().numpy())
        np.save(os.path.join(outdir, "g.npy"), g.cpu().numpy())
        np.save(os.path.join(outdir, "phi.npy"), np.array([phi]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ns,world", [(3, 2), (1, 2)])
def test_two_ranks_real_solver_equal_one_rank(tmp_path, ns, world):
    import torch
    import torch.multiprocessing as mp

    import paper_2507_10804_b200 as hv
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), ns), nprocs=world, join=True)
    wl = _case(ns)
    s = hv.Solver.from_workload(wl)
    ref = s.hessvec(wl.model, wl.probes()).astype(np.float64)
    out = np.load(tmp_path / "hv.npy")
    assert np.linalg.norm(out - ref) <= 1e-6 * np.linalg.norm(ref)
    d_obs = np.zeros((wl.ns, wl.nt, wl.nrec), np.float32)
    phi_ref, g_ref = s.gradient(wl.model, d_obs)
    assert np.linalg.norm(np.load(tmp_path / "g.npy") - g_ref) <= 1e-6 * np.linalg.norm(g_ref)
    assert abs(float(np.load(tmp_path / "phi.npy")[0]) - phi_ref) <= 1e-12 * phi_ref
