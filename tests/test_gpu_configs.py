"""The five BASELINE.json workloads at full size on the GPU.

Parity against the reference (golden sigma at sampled frequencies, made by
the reference itself) at the fp32 north-star bar, plus size-independent
properties over the whole spectrum: Parseval (sum sigma^2 = n m ||W||^2),
count n*m*min(c_in,c_out), descending order, convergence of every block,
factor quality (reconstruction, orthonormality), warm-start vs cold
agreement, the grouped one-call path (cfg4), representative-range sharding
(the multi-GPU unit of work) and the global singular-vector residual
||A v - sigma u|| with a matrix-free periodic convolution.
"""

import numpy as np
import pytest
import torch

import paper_2506_05617_b200 as cs
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.pipeline import lfa_device

from conftest import per_freq_rel_err

pytestmark = pytest.mark.gpu
TOL32 = 1e-5


def _run(layer, vectors, dev, **kw):
    w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
    return w, lfa_device(w, layer.n, layer.m, "f32", vectors, **kw)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_config_parity_and_properties(cuda, golden, cfg):
    wl = configs.WORKLOADS[cfg]
    for li, layer in enumerate(wl.layers):
        w, res = _run(layer, wl.vectors, cuda)
        info = res.info.cpu().numpy()
        assert (info > 0).all(), f"layer {li}: {np.sum(info <= 0)} blocks did not converge"
        vals = res.values.cpu().numpy()
        r = min(layer.c_out, layer.c_in)
        assert vals.shape == (layer.n * layer.m * r,)
        assert np.all(np.diff(vals) <= 0)
        w64 = configs.layer_weights(layer).astype(np.float64)
        energy = layer.n * layer.m * np.sum(w64 ** 2)
        assert abs(np.sum(vals ** 2) - energy) <= 2e-6 * energy
        key = f"cfg{cfg}_l{li}"
        if key + "_sigma" in golden.files:
            rep_of, _ = engine.partner_map(layer.n, layer.m)
            sig = res.sigma.cpu().numpy()[rep_of[golden[key + "_fidx"]]]
            assert per_freq_rel_err(sig, golden[key + "_sigma"]).max() <= TOL32, key
        if cfg == 1:
            assert np.abs(vals - golden["cfg1_l0_values"]).max() <= TOL32 * vals[0]


@pytest.mark.parametrize("cfg", [2, 5])
def test_factors_reconstruct_and_orthonormal(cuda, cfg):
    layer = configs.WORKLOADS[cfg].layers[0]
    w, res = _run(layer, True, cuda)
    blocks = engine.symbol_field(w, layer.n, layer.m, "f32", half=True)
    F_u = blocks.shape[0]
    for u in np.unique(np.linspace(0, F_u - 1, 12).astype(int)):
        A = blocks[u].cpu().numpy().astype(np.complex128)
        U = res.U[u].cpu().numpy().astype(np.complex128)
        V = res.V[u].cpu().numpy().astype(np.complex128)
        s = res.sigma[u].cpu().numpy().astype(np.float64)
        r = len(s)
        assert np.abs((U * s) @ V.conj().T - A).max() <= 1e-5 * s[0]
        assert np.abs(U.conj().T @ U - np.eye(r)).max() <= 1e-5
        assert np.abs(V.conj().T @ V - np.eye(r)).max() <= 1e-5


def test_warm_start_matches_cold(cuda):
    layer = configs.WORKLOADS[2].layers[0]
    _, cold = _run(layer, True, cuda, warm_start=False)
    _, warm = _run(layer, True, cuda, warm_start=True)
    sc, sw = cold.sigma.cpu().numpy(), warm.sigma.cpu().numpy()
    assert per_freq_rel_err(sw, sc).max() <= 2e-6
    assert warm.info.float().mean() < cold.info.float().mean()  # fewer sweeps


def test_grouped_call_equals_per_layer(cuda):
    wl = configs.WORKLOADS[4]
    blocks, single = [], []
    for layer in wl.layers[::4]:
        w = torch.from_numpy(configs.layer_weights(layer)).to(cuda)
        b = engine.symbol_field(w, layer.n, layer.m, "f32", half=True)
        blocks.append(b)
        single.append(engine.batched_svd(b, "f32", False).sigma.cpu().numpy())
    grouped = engine.batched_svd_grouped(blocks, "f32", False)
    for g, s in zip(grouped, single):
        assert np.array_equal(g.sigma.cpu().numpy(), s)
        assert (g.info.cpu().numpy() > 0).all()


def test_representative_range_shards(cuda):
    # the unit of work of one rank under frequency sharding (distributed.py)
    from paper_2506_05617_b200.distributed import shard_range

    layer = configs.WORKLOADS[2].layers[0]
    w, full = _run(layer, False, cuda)
    total = engine.half_grid_count(layer.n, layer.m)
    parts = []
    for g in range(3):
        u0, cnt = shard_range(total, g, 3)
        parts.append(lfa_device(w, layer.n, layer.m, "f32", False, u0=u0, count=cnt,
                                assemble=False).sigma.cpu().numpy())
    sh = np.concatenate(parts)
    assert per_freq_rel_err(sh, full.sigma.cpu().numpy()).max() <= 2e-6
    vals = engine.spectrum_values(torch.from_numpy(sh).to(cuda), "f32", layer.n, layer.m, True)
    assert np.abs(vals.cpu().numpy() - full.values.cpu().numpy()).max() <= 2e-6 * vals[0].item()


def _apply_periodic_conv(w, x):
    """y = A x for the unrolled periodic convolution (explicit.py:149-178 index
    layout: (x1*n + x2)*c + ch), matrix-free: y[x] = sum_{p,q} W[:,:,p,q] x[x+y(p,q)]."""
    co, ci, kh, kw = w.shape
    y = np.zeros((x.shape[0], x.shape[1], co), dtype=np.complex128)
    for p in range(kh):
        for q in range(kw):
            shifted = np.roll(x, shift=(-(p - kh // 2), -(q - kw // 2)), axis=(0, 1))
            y += shifted @ w[:, :, p, q].T
    return y


def test_global_singular_vector_residual_cfg2(cuda):
    layer = configs.WORKLOADS[2].layers[0]
    w32 = configs.layer_weights(layer)
    kernel = cs.ConvKernel.from_array(w32)
    dims = cs.SpatialDims(layer.n, layer.m)
    fld = cs.build_symbol_field(kernel, dims, return_device_tensors=True)
    res, trip = cs.spectrum_from_field(fld, values_only=False)
    smax = res.values[0]
    for f in (0, 1, 65, 2048, 4095):
        t = trip[f]
        t = cs.SvdTriplet(k=t.k, U=t.U.astype(np.complex128), sigma=t.sigma,
                          V=t.V.astype(np.complex128))
        for col in (0, 31, 63):
            v = cs.materialize_singular_vector(t, col, "right", dims).reshape(layer.m, layer.n, -1)
            u = cs.materialize_singular_vector(t, col, "left", dims)
            Av = _apply_periodic_conv(w32.astype(np.float64), v).ravel()
            assert np.linalg.norm(Av - t.sigma[col] * u) <= 1e-5 * smax


def test_device_materialize_matches_host(cuda):
    kernel = cs.random_kernel(3, 2, 3, 3, seed=18)
    dims = cs.SpatialDims(5, 4)
    fld = cs.build_symbol_field(kernel, dims, return_device_tensors=True)
    _, trip_dev = cs.spectrum_from_field(fld, values_only=False, return_device_tensors=True)
    _, trip_host = cs.spectrum_from_field(fld, values_only=False)
    for f in (0, 3, 7, 19):
        for side in ("left", "right"):
            d = cs.materialize_singular_vector(trip_dev[f], 1, side, dims).cpu().numpy()
            h = cs.materialize_singular_vector(trip_host[f], 1, side, dims)
            assert np.abs(d - h).max() <= 1e-14
    # matrix-free operator vs the dense periodic matrix at a small size
    from test_gpu_parity import _periodic_matrix

    x = (np.random.default_rng(4).standard_normal((dims.m, dims.n, 2))
         + 1j * np.random.default_rng(5).standard_normal((dims.m, dims.n, 2)))
    y = cs.apply_conv(kernel, x, dims)
    A = _periodic_matrix(kernel.weights, dims.n, dims.m)
    assert np.abs(y.ravel() - A @ x.ravel()).max() <= 1e-12


def test_global_singular_vector_residual_cfg5(cuda):
    """||A v - sigma u|| on the 16.7M x 16.7M cfg5 operator, entirely on the device."""
    layer = configs.WORKLOADS[5].layers[0]
    w, res = _run(layer, True, cuda)
    reps = engine.half_grid_indices(layer.n, layer.m)
    smax = float(res.values[0])
    for u in (0, 1, 128, 4000, 32769):
        fi, fj = divmod(int(reps[u]), layer.m)
        for col in (0, 100, 255):
            s = float(res.sigma[u, col])
            v = engine.materialize_vector(res.V[u], col, fi, fj, layer.n, layer.m, "f32")
            uu = engine.materialize_vector(res.U[u], col, fi, fj, layer.n, layer.m, "f32")
            Av = engine.apply_conv(w, v.reshape(layer.m, layer.n, -1), layer.n, layer.m, "f32")
            r = torch.linalg.vector_norm(Av.reshape(-1) - s * uu).item()
            assert r <= 1e-5 * smax, (u, col, r)


@pytest.mark.parametrize("key", ["cfg2_l0", "cfg3_l0", "cfg4_l0", "cfg4_l4", "cfg4_l8",
                                 "cfg4_l12", "cfg5_l0"])
def test_fp64_sampled_frequencies(cuda, golden, key):
    """fp64 parity mode (1e-10 per frequency) on every config's sampled
    frequencies: explicit-frequency K1 (cs_symbol_at) + fp64 Jacobi."""
    c, li = int(key[3]), int(key.split("_l")[1])
    layer = configs.WORKLOADS[c].layers[li]
    fidx = golden[key + "_fidx"]
    kernel = cs.ConvKernel.from_array(configs.layer_weights(layer).astype(np.float64))
    w = engine.weights_to_device(kernel, "f64", cuda)
    grid = cs.FrequencyGrid(cs.SpatialDims(layer.n, layer.m)).frequencies
    blocks = engine.symbol_at_freqs(w, grid[fidx], "f64")
    bn = torch.linalg.matrix_norm(blocks).cpu().numpy()
    assert np.allclose(bn, golden[key + "_blocknorm"], rtol=1e-13, atol=0)
    out = engine.batched_svd(blocks, "f64", False)
    assert (out.info.cpu().numpy() > 0).all()
    assert per_freq_rel_err(out.sigma.cpu().numpy(), golden[key + "_sigma"]).max() <= 1e-10


def test_tall_values_via_warm_vectors_matches_cold(cuda, monkeypatch):
    """cfg3 (256x128, values only) solved through the warm-started vectors
    path (engine.use_warm_values; V rows at half the X rows per lane) agrees
    with the cold values-only solve."""
    layer = configs.WORKLOADS[3].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(cuda)
    assert engine.use_warm_values(engine.half_grid_count(layer.n, layer.m), layer.c_out, layer.c_in, "f32")
    warm = lfa_device(w, layer.n, layer.m, "f32", False)
    monkeypatch.setenv("CS_WARM_VALUES", "0")
    cold = lfa_device(w, layer.n, layer.m, "f32", False)
    monkeypatch.delenv("CS_WARM_VALUES")
    assert warm.U is None and warm.V is None
    assert per_freq_rel_err(warm.sigma.cpu().numpy(), cold.sigma.cpu().numpy()).max() <= 2e-6
    assert warm.info.float().mean() < cold.info.float().mean()
