"""Multi-GPU source sharding.

Misfit, gradient and H·v are sums of independent per-source terms ("two wave equations per
source"; O10): each rank propagates a contiguous block of shots with all K probes (the probes of a shot share
one background field), the library returns rank-local partial sums, and ONE all-reduce (NCCL over
NVLink / NVSwitch on GPUs, gloo in the CPU tests) adds them. One process per GPU; torch.distributed owns the
rendezvous.
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple


def shard_range(ns: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous shot block [begin, end) of `rank`; the first ns % world ranks get one extra shot."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world / rank")
    per, extra = divmod(ns, world)
    b = rank * per + min(rank, extra)
    return b, b + per + (1 if rank < extra else 0)


def allreduce_sum(x, group=None):
    """Sum a tensor over the ranks in place (no-op when torch.distributed is not initialised)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
    return x


class ShardedOperator:
    """H·v / gradient over all shots, sharded across the ranks of a process group.

    `partial_hessvec(m, V) -> HV_local` and `partial_gradient(m, d_obs_local) -> (phi_local, g_local)` compute
    the rank's per-source partial sums (on a GPU: a `Solver` built with src_begin/src_end = shard_range(...)).
    """

    def __init__(self, partial_hessvec: Callable, partial_gradient: Optional[Callable] = None, group=None):
        self.partial_hessvec = partial_hessvec
        self.partial_gradient = partial_gradient
        self.group = group

    def hessvec(self, m, V):
        return allreduce_sum(self.partial_hessvec(m, V), self.group)

    def gradient(self, m, d_obs_local):
        import torch
        phi, g = self.partial_gradient(m, d_obs_local)
        allreduce_sum(g, self.group)
        t = torch.tensor([float(phi)], dtype=torch.float64, device=getattr(g, "device", "cpu"))
        allreduce_sum(t, self.group)
        return float(t.item()), g


def solver_operator(wl, rank: int, world: int, device: int, group=None, **solver_kw) -> ShardedOperator:
    """ShardedOperator whose partial sums run through libhv on `device` (torch CUDA tensors in and out)."""
    from . import Solver
    b, e = shard_range(wl.ns, world, rank)
    s = Solver.from_workload(wl, src_begin=b, src_end=e, device=device, **solver_kw)
    return ShardedOperator(s.hessvec, s.gradient, group)
