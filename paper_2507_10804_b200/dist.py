"""Multi-GPU sharding of the H·v / gradient / misfit sums.

Misfit, gradient and H·v are sums of independent per-source terms ("two wave equations per
source"; O10): each rank propagates a contiguous block of shots with all K probes (the probes of a shot share
one background field), the library returns rank-local partial sums, and ONE all-reduce adds them. Only when there
are fewer shots than ranks are the probes split as well (each rank then owns one shot and a contiguous block of
probe rows; the duplicated background costs 2 + 2K/G field propagations per shot instead of (2 + 2K)/G).

Two reduction paths, same result:
- torch.distributed (`allreduce_sum`): NCCL between GPUs, gloo in the CPU tests;
- in-library NCCL (`Solver.set_comm` with a communicator from `nccl_comm_create`): the library all-reduces on its
  own stream inside the call. It needs every rank to call with the SAME probe batch (no probe split), because the
  all-reduce is collective over the full [K][nz][nx] buffer.
One process per GPU; torch.distributed owns the rendezvous.
"""
from __future__ import annotations

from typing import Callable, List, NamedTuple, Optional, Tuple


def shard_range(ns: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [begin, end) of `rank`; the first ns % world ranks get one extra item (may be empty)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world / rank")
    per, extra = divmod(ns, world)
    b = rank * per + min(rank, extra)
    return b, b + per + (1 if rank < extra else 0)


class Shard(NamedTuple):
    s0: int   # shots [s0, s1)
    s1: int
    k0: int   # probe rows [k0, k1)
    k1: int
    grad: bool  # this rank contributes the gradient / misfit terms of its shots (one rank per shot)


def plan_shards(ns: int, K: int, world: int) -> List[Shard]:
    """Per-rank (shots, probe rows) covering every (shot, probe) pair exactly once.
    ns >= world: contiguous shot blocks, all K probes on every rank. ns < world: gp = world // ns probe groups per
    shot; rank r owns shot r // gp and probe block r % gp; ranks beyond ns * gp get empty shards."""
    if world < 1 or ns < 0 or K < 0:
        raise ValueError("bad sizes")
    if ns >= world:
        out = []
        for r in range(world):
            b, e = shard_range(ns, world, r)
            out.append(Shard(b, e, 0, K, True))
        return out
    gp = world // max(ns, 1)
    out = []
    for r in range(world):
        i, j = divmod(r, gp)
        if ns == 0 or i >= ns:
            out.append(Shard(ns, ns, 0, 0, False))
            continue
        k0, k1 = shard_range(K, gp, j)
        out.append(Shard(i, i + 1, k0, k1, j == 0))
    return out


def allreduce_sum(x, group=None):
    """Sum a tensor over the ranks in place (no-op when torch.distributed is not initialised)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
    return x


class ShardedOperator:
    """H·v / gradient over all shots, sharded across the ranks of a process group (the code path bench.py runs).

    `partial_hessvec(m, V_rows, out=None) -> HV_rows` computes this rank's per-source partial sums for probe rows
    V_rows over its shots (on a GPU: `Solver.hessvec` of a Solver built on `shard.s0:shard.s1`);
    `partial_gradient(m, d_obs_local) -> (phi_local, g_local)`. `in_library=True` means the partials are already
    summed over the ranks (the Solver has a NCCL communicator attached), so no torch all-reduce follows.
    """

    def __init__(self, partial_hessvec: Callable, partial_gradient: Optional[Callable] = None, group=None,
                 shard: Optional[Shard] = None, in_library: bool = False):
        self.partial_hessvec = partial_hessvec
        self.partial_gradient = partial_gradient
        self.group = group
        self.shard = shard
        self.in_library = in_library

    def _reduce(self, x):
        return x if self.in_library else allreduce_sum(x, self.group)

    def hessvec(self, m, V, out=None):
        """H [v_1..v_K] summed over all shots of all ranks; V [K][nz][nx] (every rank passes the same V)."""
        K = int(V.shape[0])
        sh = self.shard
        if sh is None or (sh.k0 == 0 and sh.k1 == K and sh.s1 > sh.s0):
            res = self.partial_hessvec(m, V, out=out) if out is not None else self.partial_hessvec(m, V)
            return self._reduce(res)
        if self.in_library:
            raise ValueError("in-library reduction needs the same probe batch on every rank (no probe split)")
        full = _zeros_like(V) if out is None else _fill0(out)
        if sh.k1 > sh.k0 and sh.s1 > sh.s0:
            full[sh.k0:sh.k1] = self.partial_hessvec(m, V[sh.k0:sh.k1])
        return allreduce_sum(full, self.group)

    def gradient(self, m, d_obs_local):
        import torch
        sh = self.shard
        if sh is None or (sh.grad and sh.s1 > sh.s0):
            phi, g = self.partial_gradient(m, d_obs_local)
        else:
            phi, g = 0.0, _zeros_like(m)
        if self.in_library:
            return float(phi), g
        allreduce_sum(g, self.group)
        t = torch.tensor([float(phi)], dtype=torch.float64, device=getattr(g, "device", "cpu"))
        allreduce_sum(t, self.group)
        return float(t.item()), g


def _zeros_like(x):
    if type(x).__module__.startswith("torch"):
        import torch
        return torch.zeros_like(x)
    import numpy as np
    return np.zeros_like(x)


def _fill0(x):
    x[...] = 0
    return x


def solver_operator(wl, rank: int, world: int, device: int, group=None, comm: Optional[int] = None,
                    **solver_kw) -> ShardedOperator:
    """ShardedOperator whose partial sums run through libhv on `device` (torch CUDA tensors in and out).
    comm: a NCCL communicator (nccl_comm_create) for in-library reduction; requires ns >= world."""
    from . import Solver
    sh = plan_shards(wl.ns, wl.n_probes, world)[rank]
    if comm is not None and wl.ns < world:
        raise ValueError("in-library NCCL reduction needs ns >= world (no probe split)")
    s = Solver.from_workload(wl, src_begin=sh.s0, src_end=sh.s1, device=device, nccl_comm=comm, **solver_kw)
    op = ShardedOperator(s.hessvec, s.gradient, group, sh, in_library=comm is not None)
    op.solver = s
    return op
