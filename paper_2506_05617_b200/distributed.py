"""Frequency-sharded LFA across the GPUs of one node.

Frequencies are independent units; rank g solves a set of conjugate-orbit
representatives with no communication during compute.  The shards are
unions of whole warm-start trees (engine.warm_forest: a cold seed and every
representative warm-started, directly or through a chain, from it), and
every kernel launch is planned for its size in the whole grid, so each
block's singular values come out bit for bit as in the single-GPU solve --
the reference's guarantee that results do not depend on the batch partition
(pkg/src/convspectra/blocksvd.py:4-8).  The one collective is an all-gather
of the per-representative singular values (NCCL over NVLink under torchrun)
when the spectrum is assembled; U/V stay sharded on their rank unless moved
to one rank by point-to-point sends.  One process per GPU; torch.distributed
is plumbing only.
"""

from __future__ import annotations

import numpy as np

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


def shard_ids(n: int, m: int, rank: int, world: int) -> np.ndarray:
    """Representative indices of `rank`'s shard: a contiguous run of whole
    warm-start trees (trees ordered by their seed's index), the runs
    balanced by representative count.  Sorted."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    level, parent, root = engine.warm_forest(n, m)
    total = len(root)
    roots, sizes = np.unique(root, return_counts=True)  # sorted by seed index
    cum = np.cumsum(sizes)
    # tree t goes to the rank whose balanced share contains its midpoint
    mid = cum - sizes / 2.0
    owner = np.minimum((mid * world / total).astype(np.int64), world - 1)
    mine = roots[owner == rank]
    return np.nonzero(np.isin(root, mine))[0].astype(np.int64)


def _all_gather_rows(rows, group=None):
    """All-gather variable-length row blocks: returns the list over ranks."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    cnt = torch.tensor([rows.shape[0]], dtype=torch.int64, device=rows.device)
    counts = [torch.empty_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    counts = [int(c.item()) for c in counts]
    cmax = max(counts)
    padded = rows.new_zeros((cmax,) + tuple(rows.shape[1:]))
    padded[: rows.shape[0]] = rows
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return [p[:c] for p, c in zip(parts, counts)]


def gather_sigma(sigma, ids, total: int, group=None):
    """All-gather per-rank sigma shards (rows of representatives `ids`) into
    the (total, r) table of every representative, on every rank."""
    import torch

    ids_t = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=sigma.device)
    all_sig = _all_gather_rows(sigma, group)
    all_ids = _all_gather_rows(ids_t, group)
    full = sigma.new_zeros((total, sigma.shape[1]))
    for s, i in zip(all_sig, all_ids):
        full[i] = s
    return full


def gather_factors(factors, ids, total: int, dst: int = 0, group=None):
    """Collect per-rank factor shards (count_g, rows, r) of representatives
    `ids` on rank ``dst``.

    SURVEY 8(e): U/V stay sharded by default; on request they move to one
    rank with grouped point-to-point sends (NCCL send/recv over NVLink under
    torchrun; an all-gather would replicate 34 GB of cfg5 factors on every
    GPU).  Complex shards travel as their real view.  Returns the
    (total, rows, r) tensor on ``dst`` and None elsewhere."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    real = torch.view_as_real(factors) if factors.is_complex() else factors
    dev = real.device
    if dist.get_backend(group) == "gloo" and real.is_cuda:
        real = real.cpu()  # gloo point-to-point moves host tensors (CPU tests)
    ids_t = torch.as_tensor(np.asarray(ids, dtype=np.int64), device=real.device)
    all_ids = _all_gather_rows(ids_t, group)  # every rank learns every shard's rows
    peer = lambda g: dist.get_global_rank(group, g) if group else g
    if rank != dst:
        dist.batch_isend_irecv([dist.P2POp(dist.isend, real.contiguous(), peer(dst), group)])[0].wait()
        return None
    out = real.new_empty((total,) + tuple(real.shape[1:]))
    bufs, ops = {}, []
    for g in range(world):
        if g == rank:
            out[all_ids[g]] = real
        elif len(all_ids[g]):
            bufs[g] = real.new_empty((len(all_ids[g]),) + tuple(real.shape[1:]))
            ops.append(dist.P2POp(dist.irecv, bufs[g], peer(g), group))
    for req in (dist.batch_isend_irecv(ops) if ops else []):
        req.wait()
    for g, b in bufs.items():
        out[all_ids[g]] = b
    out = out.to(dev)
    return torch.view_as_complex(out) if factors.is_complex() else out


def lfa_sharded(w_dev, n: int, m: int, dtype: str, want_vectors: bool = False,
                tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS,
                group=None, assemble: bool = True, timer=None,
                gather_vectors_to: int | None = None) -> DeviceSpectrum:
    """This rank's share of the LFA solve plus (optionally) the full spectrum.

    Returns the local DeviceSpectrum (sigma/U/V/info of its representatives
    ``ids``) with ``values`` holding the globally sorted spectrum when
    ``assemble``.  ``gather_vectors_to=g`` moves every rank's U/V shard to
    rank g (``gather_factors``): there U/V cover all representatives (rows in
    representative order), elsewhere None."""
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    total = engine.half_grid_count(n, m)
    if world == 1:
        return lfa_device(w_dev, n, m, dtype, want_vectors, tol, max_sweeps, assemble=assemble,
                          timer=timer)
    ids = shard_ids(n, m, rank, world)
    res = lfa_device(w_dev, n, m, dtype, want_vectors, tol, max_sweeps, ids=ids, assemble=False,
                     timer=timer)
    if gather_vectors_to is not None and want_vectors:
        res.U = gather_factors(res.U, ids, total, gather_vectors_to, group)
        res.V = gather_factors(res.V, ids, total, gather_vectors_to, group)
    if assemble:
        full = gather_sigma(res.sigma, ids, total, group)
        res.values = engine.spectrum_values(full, dtype, n, m, True)
        if timer:
            timer.mark("t3")  # assembly now includes the all-gather
    return res
