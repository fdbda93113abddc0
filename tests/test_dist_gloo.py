"""gloo tests of the multi-GPU path's host logic on CPU: contiguous shot shards, probe split
when there are fewer shots than ranks, empty shards, rank-local partial sums, one all-reduce -- through
`ShardedOperator`, the code path bench.py runs. The per-rank partial sums come from the fp64 oracle standing in
for the GPU solver (test infrastructure), so this checks the partition and the reduction, not the kernels
(tests/test_gpu_dist.py runs the real Solver through the same operator on cuda:0)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_10804_b200.dist import ShardedOperator, plan_shards, shard_range


def test_shard_range_partitions():
    for ns in range(1, 40):
        for world in range(1, 9):
            blocks = [shard_range(ns, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == ns
            for (b0, e0), (b1, e1) in zip(blocks, blocks[1:]):
                assert e0 == b1
            sizes = [e - b for b, e in blocks]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(4, 2, 2)


@pytest.mark.parametrize("ns,K,world", [(3, 2, 2), (64, 32, 8), (2, 5, 8), (2, 3, 3), (1, 1, 4), (5, 7, 4)])
def test_plan_shards_covers_every_pair_once(ns, K, world):
    cover = np.zeros((ns, K), dtype=int)
    grad = np.zeros(ns, dtype=int)
    for sh in plan_shards(ns, K, world):
        cover[sh.s0:sh.s1, sh.k0:sh.k1] += 1
        if sh.grad:
            grad[sh.s0:sh.s1] += 1
    assert np.all(cover == 1) and np.all(grad == 1)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(ns):
    import workloads as W
    return W.custom(10, 14, nt=60, W=6, ns=ns, n_probes=3, f_peak=20.0, seed=4)


def _worker(rank, world, port, outdir, ns):
    from oracle import wave
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    wl = _case(ns)
    pb = wave.Problem(wl)
    sh = plan_shards(wl.ns, wl.n_probes, world)[rank]
    b, e = sh.s0, sh.s1
    V = wl.probes().astype(np.float64)
    d_obs = wave.Problem(wl, wl.model_true).forward_all()

    def partial_hessvec(m, Vt):
        return torch.from_numpy(pb.hessvec(list(Vt.numpy()), shots=range(b, e)))

    def partial_gradient(m, dloc):
        phi, g = pb.gradient(dloc, shots=range(b, e))
        return phi, torch.from_numpy(g)

    op = ShardedOperator(partial_hessvec, partial_gradient, shard=sh)
    HV = op.hessvec(torch.zeros(wl.nz, wl.nx, dtype=torch.float64), torch.from_numpy(V))
    phi, g = op.gradient(torch.zeros(wl.nz, wl.nx, dtype=torch.float64), d_obs[b:e])
    if rank == 0:
        np.save(os.path.join(outdir, "hv.npy"), HV.numpy())
        np.save(os.path.join(outdir, "g.npy"), g.numpy())
        np.save(os.path.join(outdir, "phi.npy"), np.array([phi]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("ns,world", [(3, 2), (1, 2)])
def test_two_rank_gloo_sum_equals_single_process(tmp_path, ns, world):
    """(3 shots, 2 ranks): shot shards; (1 shot, 2 ranks): probe split (rank 0 rows 0-1, rank 1 row 2)."""
    from oracle import wave
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path), ns), nprocs=world, join=True)
    wl = _case(ns)
    pb = wave.Problem(wl)
    ref = pb.hessvec(list(wl.probes().astype(np.float64)))
    d_obs = wave.Problem(wl, wl.model_true).forward_all()
    phi_ref, g_ref = pb.gradient(d_obs)
    hv = np.load(tmp_path / "hv.npy")
    assert np.linalg.norm(hv - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(np.load(tmp_path / "g.npy") - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
    assert abs(float(np.load(tmp_path / "phi.npy")[0]) - phi_ref) <= 1e-12 * phi_ref
