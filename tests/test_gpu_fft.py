"""FFT route to the symbol field (csrc/cs_fft.cu): the
reference's fft.py tests (pkg/tests/test_fft.py:58-105) through this
package's API, plus cross-checks against K1 and the goldens."""

import numpy as np
import pytest
import torch

import paper_2506_05617_b200 as cs
from paper_2506_05617_b200 import configs, engine
from conftest import per_freq_rel_err

pytestmark = pytest.mark.gpu


def identity_kernel(channels):
    w = np.zeros((channels, channels, 1, 1))
    w[:, :, 0, 0] = np.eye(channels)
    return cs.ConvKernel.from_array(w)


def test_identity_kernel_field_matches_symbol_path(cuda):
    dims = cs.SpatialDims(4, 4)
    via_fft = cs.fft_symbol_field(identity_kernel(2), dims)
    via_sym = cs.build_symbol_field(identity_kernel(2), dims)
    assert via_fft.blocks.shape == (16, 2, 2)
    assert np.allclose(via_fft.blocks, np.eye(2), atol=1e-13)
    assert np.allclose(via_fft.blocks, via_sym.blocks, atol=1e-13)
    assert via_fft.source == "fft"


def test_averaging_2x2_wrapped_scalars(cuda):
    # kernel wider than the torus: taps wrap and accumulate (fft.py:136-138)
    k = cs.ConvKernel.from_array(np.full((1, 1, 3, 3), 1.0 / 9.0))
    fld = cs.fft_symbol_field(k, cs.SpatialDims(2, 2))
    got = np.sort(fld.blocks[:, 0, 0].real)
    assert np.allclose(got, [-1 / 3, -1 / 3, 1 / 9, 1.0], atol=1e-13)


@pytest.mark.parametrize("n,m,co,ci,kh,kw,seed", [(6, 4, 2, 2, 3, 3, 21), (5, 7, 3, 2, 3, 3, 22),
                                                  (2, 3, 2, 3, 5, 5, 23), (16, 12, 8, 4, 5, 3, 24)])
def test_blocks_match_symbol_path_f64(cuda, n, m, co, ci, kh, kw, seed):
    kernel = cs.random_kernel(co, ci, kh, kw, seed=seed)
    dims = cs.SpatialDims(n=n, m=m)
    a = cs.fft_symbol_field(kernel, dims).blocks
    b = cs.build_symbol_field(kernel, dims).blocks
    assert np.abs(a - b).max() <= 1e-12 * np.abs(b).max()


@pytest.mark.parametrize("dims,channels,seed", [((8, 8), (3, 3), 22), ((6, 10), (2, 3), 23),
                                                ((5, 5), (1, 1), 24)])
def test_cross_path_spectra(cuda, dims, channels, seed):
    kernel = cs.random_kernel(channels[1], channels[0], 3, 3, seed=seed)
    sd = cs.SpatialDims(*dims)
    lfa = cs.compute_spectrum(kernel, sd, method="lfa").values
    res = cs.compute_spectrum(kernel, sd, method="fft")
    assert res.method == "fft"
    assert np.allclose(res.values, lfa, rtol=1e-8, atol=1e-12 * lfa[0])


def test_fft_timing_split(cuda):
    fld = cs.fft_symbol_field(cs.random_kernel(2, 2, 3, 3, seed=25), cs.SpatialDims(8, 8))
    assert fld.s_transform > 0 and fld.s_copy > 0
    res = cs.compute_spectrum(cs.random_kernel(2, 2, 3, 3, seed=25), cs.SpatialDims(8, 8), method="fft")
    assert res.timings.s_transform > 0 and res.timings.s_copy > 0 and res.timings.s_svd > 0


@pytest.mark.parametrize("cfg", [1, 2])
def test_fft_route_half_grid_f32_matches_k1_and_goldens(cuda, golden, cfg):
    """fp32 half-grid representatives from the FFT route vs K1 (rounding
    level of the field), then the spectrum at the north-star bar vs golden."""
    layer = configs.WORKLOADS[cfg].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(cuda)
    a = engine.fft_symbol_field(w, layer.n, layer.m, "f32", half=True)
    b = engine.symbol_field(w, layer.n, layer.m, "f32", half=True)
    scale = b.abs().amax(dim=(1, 2), keepdim=True)
    assert ((a - b).abs() / scale).max().item() <= 2e-6
    from paper_2506_05617_b200.pipeline import lfa_device
    res = lfa_device(w, layer.n, layer.m, "f32", False, method="fft")
    key = f"cfg{cfg}_l0"
    rep_of, _ = engine.partner_map(layer.n, layer.m)
    sig = res.sigma.cpu().numpy()[rep_of[golden[key + "_fidx"]]]
    assert per_freq_rel_err(sig, golden[key + "_sigma"]).max() <= 1e-5


def test_fft_budget_and_explicit_refused(cuda):
    with pytest.raises(cs.AllocationFailure):
        cs.fft_symbol_field(cs.random_kernel(64, 64, 3, 3), cs.SpatialDims(64, 64), mem_budget_gib=0.01)
    with pytest.raises(NotImplementedError):
        cs.compute_spectrum(cs.random_kernel(2, 2, 3, 3), cs.SpatialDims(4, 4), method="explicit")


def test_fft_route_cfg5_field_matches_k1(cuda):
    """Full-size FFT route (cfg5: 65536 channel pairs x 2^16-point DFTs, 2^32
    points, 64-bit cuFFT plan) against K1 on every representative block."""
    layer = configs.WORKLOADS[5].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(cuda)
    a = engine.fft_symbol_field(w, layer.n, layer.m, "f32", half=True)
    b = engine.symbol_field(w, layer.n, layer.m, "f32", half=True)
    assert a.shape == b.shape == (engine.half_grid_count(layer.n, layer.m), 256, 256)
    worst = 0.0
    for s in range(0, a.shape[0], 4096):  # chunked: the difference of 17 GB fields
        d = (a[s:s + 4096] - b[s:s + 4096]).abs().amax(dim=(1, 2))
        ref = b[s:s + 4096].abs().amax(dim=(1, 2))
        worst = max(worst, (d / ref).max().item())
    assert worst <= 2e-6
