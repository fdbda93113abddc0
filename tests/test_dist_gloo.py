"""World-size-2 gloo test of the multi-GPU path's host logic on CPU: contiguous shot shards,
rank-local partial sums, one all-reduce. The per-rank partial sums come from the fp64 oracle standing in for
the GPU solver (test infrastructure), so this checks the partition and the reduction, not the kernels."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_10804_b200.dist import ShardedOperator, shard_range


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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    import workloads as W
    from oracle import wave
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    wl = W.custom(10, 14, nt=60, W=6, ns=3, n_probes=2, f_peak=20.0, seed=4)
    pb = wave.Problem(wl)
    b, e = shard_range(wl.ns, world, rank)
    V = wl.probes().astype(np.float64)
    d_obs = wave.Problem(wl, wl.model_true).forward_all()

    def partial_hessvec(m, Vt):
        return torch.from_numpy(pb.hessvec(list(Vt.numpy()), shots=range(b, e)))

    def partial_gradient(m, dloc):
        phi, g = pb.gradient(dloc, shots=range(b, e))
        return phi, torch.from_numpy(g)

    op = ShardedOperator(partial_hessvec, partial_gradient)
    HV = op.hessvec(None, torch.from_numpy(V))
    phi, g = op.gradient(None, d_obs[b:e])
    if rank == 0:
        np.save(os.path.join(outdir, "hv.npy"), HV.numpy())
        np.save(os.path.join(outdir, "g.npy"), g.numpy())
        np.save(os.path.join(outdir, "phi.npy"), np.array([phi]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sum_equals_single_process(tmp_path):
    import workloads as W
    from oracle import wave
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    wl = W.custom(10, 14, nt=60, W=6, ns=3, n_probes=2, f_peak=20.0, seed=4)
    pb = wave.Problem(wl)
    ref = pb.hessvec(list(wl.probes().astype(np.float64)))
    d_obs = wave.Problem(wl, wl.model_true).forward_all()
    phi_ref, g_ref = pb.gradient(d_obs)
    hv = np.load(tmp_path / "hv.npy")
    assert np.linalg.norm(hv - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.linalg.norm(np.load(tmp_path / "g.npy") - g_ref) <= 1e-12 * np.linalg.norm(g_ref)
    assert abs(float(np.load(tmp_path / "phi.npy")[0]) - phi_ref) <= 1e-12 * phi_ref
