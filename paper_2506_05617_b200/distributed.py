"""Frequency-sharded LFA across the GPUs of one node.

Frequencies are independent units: rank g solves the contiguous range of
conjugate-orbit representatives ``shard_range(F_u, g, G)`` with no
communication during compute.  The one collective is an all-gather of the
per-representative singular values (NCCL over NVLink under torchrun) when
the spectrum is assembled; U/V stay sharded on their rank.  One process per
GPU; torch.distributed is plumbing only.
"""

from __future__ import annotations

from . import engine
from .engine import DEFAULT_MAX_SWEEPS, DEFAULT_SVD_TOL
from .pipeline import DeviceSpectrum, lfa_device


def shard_range(total: int, rank: int, world: int):
    """Contiguous, balanced split of [0, total): (start, count) of `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_sigma(sigma, total: int, group=None):
    """All-gather per-rank (count_g, r) sigma shards into (total, r) in rank order.

    Shards are padded to the largest count so the collective is uniform."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r = sigma.shape[1]
    counts = [shard_range(total, g, world)[1] for g in range(world)]
    cmax = max(counts)
    padded = sigma.new_zeros((cmax, r))
    padded[: sigma.shape[0]] = sigma
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    assert counts[rank] == sigma.shape[0]
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def lfa_sharded(w_dev, n: int, m: int, dtype: str, want_vectors: bool = False,
                tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS,
                group=None, assemble: bool = True, timer=None) -> DeviceSpectrum:
    """This rank's share of the LFA solve plus (optionally) the full spectrum.

    Returns the local DeviceSpectrum (sigma/U/V/info of its representatives)
    with ``values`` holding the globally sorted spectrum when ``assemble``."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    total = engine.half_grid_count(n, m)
    u0, cnt = shard_range(total, rank, world)
    res = lfa_device(w_dev, n, m, dtype, want_vectors, tol, max_sweeps, u0=u0, count=cnt,
                     assemble=(world == 1 and assemble), timer=timer)
    if world > 1 and assemble:
        full = gather_sigma(res.sigma, total, group)
        res.values = engine.spectrum_values(full, dtype, n, m, True)
        if timer:
            timer.mark("t3")  # assembly now includes the all-gather
    return res
