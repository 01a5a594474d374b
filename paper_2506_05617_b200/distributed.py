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


def gather_factors(factors, total: int, dst: int = 0, group=None):
    """Collect per-rank factor shards (count_g, rows, r) on rank ``dst``.

    SURVEY 8(e): U/V stay sharded by default; on request they move to one
    rank with grouped point-to-point sends (NCCL send/recv over NVLink under
    torchrun; an all-gather would replicate 34 GB of cfg5 factors on every
    GPU).  Complex shards travel as their real view.  Returns the
    (total, rows, r) tensor on ``dst`` and None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    spans = [shard_range(total, g, world) for g in range(world)]
    assert factors.shape[0] == spans[rank][1]
    real = torch.view_as_real(factors) if factors.is_complex() else factors
    dev = real.device
    if dist.get_backend(group) == "gloo" and real.is_cuda:
        real = real.cpu()  # gloo point-to-point moves host tensors (CPU tests)
    if rank != dst:
        dist.batch_isend_irecv([dist.P2POp(dist.isend, real.contiguous(),
                                           dist.get_global_rank(group, dst) if group else dst,
                                           group)])[0].wait()
        return None
    out = real.new_empty((total,) + tuple(real.shape[1:]))
    ops = []
    for g, (u0, cnt) in enumerate(spans):
        if g == rank:
            out[u0:u0 + cnt] = real
        elif cnt:
            ops.append(dist.P2POp(dist.irecv, out[u0:u0 + cnt],
                                  dist.get_global_rank(group, g) if group else g, group))
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    out = out.to(dev)
    return torch.view_as_complex(out) if factors.is_complex() else out


def lfa_sharded(w_dev, n: int, m: int, dtype: str, want_vectors: bool = False,
                tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS,
                group=None, assemble: bool = True, timer=None,
                gather_vectors_to: int | None = None) -> DeviceSpectrum:
    """This rank's share of the LFA solve plus (optionally) the full spectrum.

    Returns the local DeviceSpectrum (sigma/U/V/info of its representatives)
    with ``values`` holding the globally sorted spectrum when ``assemble``.
    ``gather_vectors_to=g`` moves every rank's U/V shard to rank g
    (``gather_factors``): there U/V cover all representatives, elsewhere None."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    total = engine.half_grid_count(n, m)
    u0, cnt = shard_range(total, rank, world)
    res = lfa_device(w_dev, n, m, dtype, want_vectors, tol, max_sweeps, u0=u0, count=cnt,
                     assemble=(world == 1 and assemble), timer=timer)
    if world > 1 and gather_vectors_to is not None and want_vectors:
        res.U = gather_factors(res.U, total, gather_vectors_to, group)
        res.V = gather_factors(res.V, total, gather_vectors_to, group)
    if world > 1 and assemble:
        full = gather_sigma(res.sigma, total, group)
        res.values = engine.spectrum_values(full, dtype, n, m, True)
        if timer:
            timer.mark("t3")  # assembly now includes the all-gather
    return res
