"""Frequency sharding host logic on CPU: world_size 2 over gloo.

The GPU path (lfa_sharded) adds only the device solve per shard; here the
partition and the sigma all-gather + assembly order are checked with CPU
tensors (the collective is the same torch.distributed call NCCL runs)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2506_05617_b200 import engine
from paper_2506_05617_b200.distributed import gather_factors, gather_sigma, shard_ids, shard_range


@pytest.mark.parametrize("total", [1, 7, 514, 32770])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_range_partitions(total, world):
    spans = [shard_range(total, g, world) for g in range(world)]
    assert spans[0][0] == 0
    for (s0, c0), (s1, _) in zip(spans, spans[1:]):
        assert s0 + c0 == s1
    assert sum(c for _, c in spans) == total
    counts = [c for _, c in spans]
    assert max(counts) - min(counts) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, m, r, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    total = engine.half_grid_count(n, m)
    ids = shard_ids(n, m, rank, world)
    # each rank "solves" its representatives: sigma row u = [u, u/2, ...]
    sig = torch.stack([torch.as_tensor(ids, dtype=torch.float64) / (j + 1) for j in range(r)], dim=1)
    full = gather_sigma(sig, ids, total)
    if rank == 0:
        q.put(full.numpy())
    dist.destroy_process_group()


def test_gather_sigma_world2_gloo():
    n, m, r = 7, 6, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, 2, port, n, m, r, q)) for g in range(2)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = engine.half_grid_count(n, m)
    expect = np.stack([np.arange(total) / (j + 1) for j in range(r)], axis=1)
    assert np.array_equal(full, expect)
    # spectrum assembly rule: every non-self-conjugate representative twice
    rep_of, _ = engine.partner_map(n, m)
    values = np.sort(full[rep_of].ravel())[::-1]
    assert len(values) == n * m * r


def _factor_worker(rank, world, port, total, rows, r, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ids = np.array([u for u in range(total) if u % world == rank], dtype=np.int64)  # any row set
    cnt = len(ids)
    # shard u of the factor: entries u + 1j * (row * r + col)
    idx = torch.as_tensor(ids, dtype=torch.float32)[:, None, None]
    im = torch.arange(rows * r, dtype=torch.float32).reshape(1, rows, r)
    shard = torch.complex(idx.expand(cnt, rows, r), im.expand(cnt, rows, r)).contiguous()
    full = gather_factors(shard, ids, total, dst=world - 1)
    if rank == world - 1:
        q.put(full.numpy())
    else:
        assert full is None
    dist.destroy_process_group()


@pytest.mark.parametrize("n,m,world", [(64, 64, 2), (64, 64, 3), (256, 256, 8), (7, 6, 2), (56, 56, 4)])
def test_shard_ids_are_whole_trees(n, m, world):
    """Shards partition the representatives into whole warm-start trees
    (every parent in the same shard), balanced within one tree's size."""
    level, parent, root = engine.warm_forest(n, m)
    total = engine.half_grid_count(n, m)
    shards = [shard_ids(n, m, g, world) for g in range(world)]
    allids = np.concatenate(shards)
    assert np.array_equal(np.sort(allids), np.arange(total))
    biggest = np.bincount(root).max()
    for ids in shards:
        assert np.all(np.diff(ids) > 0)
        par = parent[ids]
        assert np.isin(par[par >= 0], ids).all()
        assert abs(len(ids) - total / world) <= biggest
    # plans restricted to a shard are the global plan's stages (sizes from the whole grid)
    for ids in shards:
        stages = engine.subset_plan(n, m, ids, "cpu")
        got = sum(len(s[0]) for s in stages)
        assert got == len(ids)
        for sel, pred, gsize in stages:
            assert gsize == np.count_nonzero(level == level[ids[sel.numpy()[0]]])


@pytest.mark.parametrize("world,total", [(2, 11), (3, 10)])
def test_gather_factors_to_one_rank_gloo(world, total):
    """U/V shards to one rank by grouped point-to-point sends."""
    rows, r = 4, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_factor_worker, args=(g, world, port, total, rows, r, q))
             for g in range(world)]
    for p in procs:
        p.start()
    full = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert full.shape == (total, rows, r)
    assert np.array_equal(full.real, np.broadcast_to(np.arange(total)[:, None, None], (total, rows, r)))
    assert np.array_equal(full.imag, np.broadcast_to(np.arange(rows * r).reshape(1, rows, r), (total, rows, r)))
