"""Frequency-sharded solve (distributed.lfa_sharded) with 2 and 3 ranks on one GPU.

The only GPU available to this run is cuda:0, so every rank uses it and the
sigma all-gather runs over gloo (host-mediated).  Nothing on the device waits
for another rank: each rank solves its own shard (whole warm-start trees),
then the collective exchanges the sigma shards -- the same code path NCCL
runs on a multi-GPU node.  The reference guarantees results independent of
the batch partition (blocksvd.py:4-8, T/test_acceptance.py:139-146): the
assembled spectrum and every shard's sigma must equal the single-rank solve
BIT FOR BIT.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cfg, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2506_05617_b200 import configs
    from paper_2506_05617_b200.distributed import lfa_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    layer = configs.WORKLOADS[cfg].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).cuda()
    res = lfa_sharded(w, layer.n, layer.m, "f32", configs.WORKLOADS[cfg].vectors)
    q.put((rank, res.ids, res.values.cpu().numpy(), res.sigma.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world", [(1, 2), (2, 2), (2, 3), (3, 2)])
def test_shards_match_single_bitwise(cuda, cfg, world):
    from paper_2506_05617_b200 import configs
    from paper_2506_05617_b200.pipeline import lfa_device

    layer = configs.WORKLOADS[cfg].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(cuda)
    single = lfa_device(w, layer.n, layer.m, "f32", configs.WORKLOADS[cfg].vectors)
    ref_vals = single.values.cpu().numpy()
    ref_sig = single.sigma.cpu().numpy()

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(g, world, port, cfg, q)) for g in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o[0])
    covered = np.sort(np.concatenate([o[1] for o in outs]))
    assert np.array_equal(covered, np.arange(len(ref_sig)))
    for _, ids, vals, sig in outs:
        assert np.array_equal(vals, ref_vals)
        assert np.array_equal(sig, ref_sig[ids])


def _vec_worker(rank, world, port, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist

    from paper_2506_05617_b200 import configs, engine
    from paper_2506_05617_b200.distributed import gather_sigma, lfa_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    layer = configs.WORKLOADS[2].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).cuda()
    res = lfa_sharded(w, layer.n, layer.m, "f32", True, gather_vectors_to=1)
    full = gather_sigma(res.sigma, res.ids, engine.half_grid_count(layer.n, layer.m))
    if rank == 1:
        blocks = engine.symbol_field(w, layer.n, layer.m, "f32", half=True)
        F_u = blocks.shape[0]
        worst = 0.0
        for u in np.unique(np.linspace(0, F_u - 1, 16).astype(int)):
            A = blocks[u].cpu().numpy().astype(np.complex128)
            U = res.U[u].cpu().numpy().astype(np.complex128)
            V = res.V[u].cpu().numpy().astype(np.complex128)
            s = full[u].cpu().numpy().astype(np.float64)
            worst = max(worst, np.abs((U * s) @ V.conj().T - A).max() / s[0])
        q.put((res.U.shape[0], F_u, worst))
    else:
        q.put((res.U is None, res.V is None, 0.0))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gather_vectors_to_one_rank(cuda):
    """U/V shards moved to one rank (distributed.gather_factors) reconstruct
    every sampled block with the all-gathered sigma."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_vec_worker, args=(g, 2, port, q)) for g in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for a, b, worst in outs:
        if a is True:
            assert b is True  # rank 0 keeps nothing
        else:
            assert a == b and worst <= 1e-5
