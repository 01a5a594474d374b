"""Dense parity pins where the warm-started device solver acts (round 2).

Goldens: tests/golden/golden_deep.npz, made by the reference itself
(make_golden_deep.py: _symbol_blocks + _svd_values_batch, f64, tol 1e-13).

* cfg5 at 259 frequencies: the 4 self-conjugate ones, 64 from the deepest
  stages (BFS level >= 12) of the depth-8 warm-start forest, 191 random --
  fp32 (tensor-core blocked Jacobi on the warm stages) at 1e-5 and fp64 at
  1e-10, plus V orthonormality of the deepest-chain frequencies;
* cfg2 on the full representative set, fp32 (1e-5) and fp64 (1e-10);
* all four 256^2 and all four 512^2 ResNet-18 layers of cfg4 on every
  representative, through the one-call grouped path;
* the reference's values_only invariant, bitwise, on cfg2.
Bar: per frequency max_j |sigma - sigma_ref| / sigma_ref[0] (north_star).
"""

import os

import numpy as np
import pytest
import torch

import paper_2506_05617_b200 as cs
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.pipeline import lfa_device, lfa_device_multi

from conftest import per_freq_rel_err

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def deep():
    return np.load(os.path.join(HERE, "golden", "golden_deep.npz"))


def _w(layer, dev, dtype):
    w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
    return w if dtype == "f32" else w.double()


@pytest.mark.parametrize("dtype,bar", [("f32", 1e-5), ("f64", 1e-10)])
def test_cfg5_deep_frequencies(cuda, deep, dtype, bar):
    layer = configs.WORKLOADS[5].layers[0]
    res = lfa_device(_w(layer, cuda, dtype), layer.n, layer.m, dtype, True)
    assert (res.info.cpu().numpy() > 0).all()
    rep_of, conj = engine.partner_map(layer.n, layer.m)
    fidx = deep["cfg5_deep_fidx"]
    u = rep_of[fidx]
    sig = res.sigma[torch.from_numpy(u).to(cuda)].cpu().numpy().astype(np.float64)
    err = per_freq_rel_err(sig, deep["cfg5_deep_sigma"])
    assert err.max() <= bar, (dtype, err.max(), fidx[err.argmax()])
    # deepest warm chains: right factors stay orthonormal
    stage = deep["cfg5_deep_stage"]
    sel = u[np.argsort(-stage)[:16]]
    V = res.V[torch.from_numpy(sel).to(cuda)].cpu().numpy().astype(np.complex128)
    orth = max(np.abs(v.conj().T @ v - np.eye(v.shape[1])).max() for v in V)
    assert orth <= (1e-5 if dtype == "f32" else 1e-10), orth


@pytest.mark.parametrize("dtype,bar", [("f32", 1e-5), ("f64", 1e-10)])
def test_cfg2_full_grid(cuda, deep, dtype, bar):
    layer = configs.WORKLOADS[2].layers[0]
    res = lfa_device(_w(layer, cuda, dtype), layer.n, layer.m, dtype, True)
    sig = res.sigma.cpu().numpy().astype(np.float64)
    err = per_freq_rel_err(sig, deep["cfg2_full_sigma"])
    assert err.max() <= bar, (dtype, err.max())
    V = res.V.cpu().numpy().astype(np.complex128)
    orth = np.abs(np.einsum("fij,fik->fjk", V.conj(), V) - np.eye(V.shape[2])).max()
    assert orth <= (1e-5 if dtype == "f32" else 1e-10), orth


def test_cfg4_every_large_layer_grouped(cuda, deep):
    """All 16 layers in one grouped call; every representative of the eight
    256^2 / 512^2 layers against the reference."""
    wl = configs.WORKLOADS[4]
    layers = [(_w(l, cuda, "f32"), l.n, l.m) for l in wl.layers]
    outs = lfa_device_multi(layers, "f32", False)
    checked = 0
    for li, (l, o) in enumerate(zip(wl.layers, outs)):
        key = f"cfg4_l{li}_full_sigma"
        if key not in deep.files:
            continue
        err = per_freq_rel_err(o.sigma.cpu().numpy().astype(np.float64), deep[key])
        assert err.max() <= 1e-5, (li, err.max())
        checked += 1
    assert checked == 8


def test_values_only_bitwise_cfg2(cuda):
    """The reference returns identical values with and without vectors
    (pipeline.py:40-42, T/test_blocksvd.py:110-116); so does the drop-in."""
    layer = configs.WORKLOADS[2].layers[0]
    k = cs.ConvKernel.from_array(configs.layer_weights(layer))
    dims = cs.SpatialDims(layer.n, layer.m)
    for dt in ("f32", "f64"):
        a = cs.compute_spectrum(k, dims, values_only=True, dtype=dt).values
        b = cs.compute_spectrum(k, dims, values_only=False, dtype=dt).values
        assert np.array_equal(a, b), dt


def test_cfg5_lazy_partner_triplets(cuda):
    """spectrum_from_field(values_only=False) on the full cfg5 field (65,536
    blocks of 256 x 256) keeps the half-grid factors on the device and
    materialises a frequency's triplet on access -- partners by conjugation
    (blocksvd.py:271-275 returns views; the expanded fp32 grid alone would
    be 2 x 34 GB more)."""
    layer = configs.WORKLOADS[5].layers[0]
    k = cs.ConvKernel.from_array(configs.layer_weights(layer))
    dims = cs.SpatialDims(layer.n, layer.m)
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats(cuda)
    fld = cs.build_symbol_field(k, dims, dtype="f32", return_device_tensors=True)
    res, trip = cs.spectrum_from_field(fld, values_only=False, return_device_tensors=True)
    assert len(trip) == layer.n * layer.m
    peak = torch.cuda.max_memory_allocated(cuda)
    field = fld.blocks.numel() * 8
    assert peak <= field + 2.2 * field / 2 + field / 2 + (8 << 30), peak  # field + U/V + reps, no expansion
    smax = res.values[0]
    rep_of, conj = engine.partner_map(layer.n, layer.m)
    fs = [0, 1, 255, 256 * 129 + 7]
    fs += [int(np.nonzero(rep_of == rep_of[f])[0][-1]) for f in fs]  # partners
    for f in fs:
        t = trip[f]
        A = fld.blocks[f].cpu().numpy().astype(np.complex128)
        U, V = t.U.cpu().numpy().astype(np.complex128), t.V.cpu().numpy().astype(np.complex128)
        s = t.sigma.cpu().numpy().astype(np.float64)
        assert np.abs((U * s) @ V.conj().T - A).max() <= 1e-5 * smax, f
    host = cs.spectrum_from_field  # host-typed access: one block copied per item
    del trip
    _, trip_h = host(fld, values_only=False)
    t = trip_h[fs[-1]]
    assert isinstance(t.U, np.ndarray) and t.U.dtype == np.complex128 and t.U.shape == (256, 256)


def test_tensor_core_kernel_matches_scalar_kernel(cuda, monkeypatch):
    """K3 (tensor-core blocked Jacobi: TMEM-fed, warp-specialised update)
    against K2 (scalar panel kernel, CS_TCB=0) on the same warm-started cfg5
    blocks: sigma within 2e-6 of sigma_max, the energy identity
    sum sigma^2 = ||A||_F^2, orthonormal U / V and A V = U diag(sigma)
    (CS/blocksvd.py:155-173 is what both replace)."""
    layer = configs.WORKLOADS[5].layers[0]
    w = _w(layer, cuda, "f32")
    count = 1024  # four full rows of the half grid (whole warm-start trees; seven rounds of the work queue)
    k3 = lfa_device(w, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=True, assemble=False)
    monkeypatch.setenv("CS_TCB", "0")
    k2 = lfa_device(w, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=True, assemble=False)
    monkeypatch.delenv("CS_TCB")
    assert (k3.info > 0).all() and (k2.info > 0).all()
    s3, s2 = k3.sigma.cpu().numpy(), k2.sigma.cpu().numpy()
    assert per_freq_rel_err(s3, s2).max() <= 2e-6
    A = engine.symbol_field(w, layer.n, layer.m, "f32", half=True, f_first=0, f_count=count)
    fro = (A.abs().double() ** 2).sum(dim=(1, 2)).cpu().numpy()
    energy = np.abs((s3.astype(np.float64) ** 2).sum(axis=1) - fro) / fro
    assert energy.max() <= 5e-6
    eye = torch.eye(layer.c_in, device=cuda, dtype=torch.complex64)
    for F in (k3.U, k3.V):
        assert (F.mH @ F - eye).abs().amax().item() <= 2e-5
    res = (A @ k3.V - k3.U * k3.sigma[:, None, :].to(torch.complex64)).abs().amax(dim=(1, 2))
    assert (res / k3.sigma[:, 0]).max().item() <= 2e-5
