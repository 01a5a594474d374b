"""The CPU oracle (oracle/oracle.c) against vectors produced by the reference
itself (tests/golden/make_golden.py imports conv-spectra 0.1.0).  CPU only.

The oracle is bit-exact with the reference's numba kernels on this container
(same operation order, no FMA contraction); across hosts libm may differ in
the last ulp, so comparisons allow a few ulps.
"""

import hashlib

import numpy as np
import pytest

from paper_2506_05617_b200 import configs

from conftest import per_freq_rel_err


@pytest.mark.parametrize("name", ["a", "b", "c", "d"])
def test_symbol_blocks_match_reference(golden, orc, name):
    co, ci, kh, kw, seed, n, m = (int(v) for v in golden[f"sym_{name}_shape"])
    rng = np.random.Generator(np.random.Philox(key=seed))
    w = rng.standard_normal((co, ci, kh, kw))
    got = orc.symbol_field(w, n, m)
    ref = golden[f"sym_{name}_blocks"]
    assert got.shape == ref.shape
    assert np.abs(got - ref).max() <= 1e-15 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("idx", range(4))
def test_fixture_spectra_match_reference(golden, orc, idx):
    n, m, c_in, c_out, seed = (int(v) for v in golden[f"fix{idx}_shape"])
    rng = np.random.Generator(np.random.Philox(key=seed))
    w = rng.standard_normal((c_out, c_in, 3, 3))
    vals = orc.spectrum_values(w, n, m)
    ref = golden[f"fix{idx}_values"]
    assert np.abs(vals - ref).max() <= 1e-13 * ref[0]
    # per-frequency sigma through the vectors path
    U, sig, V, fail = orc.svd_full(orc.symbol_field(w, n, m))
    assert not fail.any()
    assert per_freq_rel_err(sig, golden[f"fix{idx}_sigma"]).max() <= 1e-13
    assert np.allclose(vals, golden[f"fix{idx}_dense"], rtol=1e-6, atol=0)


def test_cfg1_complete(golden, orc):
    layer = configs.WORKLOADS[1].layers[0]
    w = configs.layer_weights(layer).astype(np.float64)
    vals = orc.spectrum_values(w, layer.n, layer.m)
    ref = golden["cfg1_l0_values"]
    assert vals.shape == (16 * 1024,)
    assert np.abs(vals - ref).max() <= 1e-13 * ref[0]


@pytest.mark.parametrize("cfg,layer_idx,maxf", [(2, 0, 16), (3, 0, 8), (4, 0, 8), (4, 4, 8),
                                                (4, 8, 4), (5, 0, 4)])
def test_sampled_config_sigma(golden, orc, cfg, layer_idx, maxf):
    layer = configs.WORKLOADS[cfg].layers[layer_idx]
    key = f"cfg{cfg}_l{layer_idx}"
    fidx = golden[key + "_fidx"][:maxf]
    w = configs.layer_weights(layer).astype(np.float64)
    freqs = orc.grid_frequencies(layer.n, layer.m)[fidx]
    blocks = orc.symbol_field(w, freqs=freqs)
    assert np.allclose(np.linalg.norm(blocks, axis=(1, 2)), golden[key + "_blocknorm"][:maxf],
                       rtol=1e-14, atol=0)
    sig, fail = orc.svd_values(blocks)
    assert not fail.any()
    assert per_freq_rel_err(sig, golden[key + "_sigma"][:maxf]).max() <= 1e-12


@pytest.mark.parametrize("i", range(8))
def test_svd_block_triplets(golden, orc, i):
    A = golden[f"blk{i}_A"]
    U, sig, V, fail = orc.svd_full(A[None])
    assert np.abs(sig[0] - golden[f"blk{i}_sigma"]).max() <= 1e-13 * golden[f"blk{i}_sigma"][0]
    # factors are unique up to a unit phase per column: compare projectors U_j U_j^H
    for j in range(len(sig[0])):
        a = np.outer(U[0][:, j], U[0][:, j].conj())
        b = np.outer(golden[f"blk{i}_U"][:, j], golden[f"blk{i}_U"][:, j].conj())
        assert np.abs(a - b).max() <= 1e-9


def test_weights_generator_pinned(golden):
    for c, wl in configs.WORKLOADS.items():
        for li, layer in enumerate(wl.layers):
            digest = hashlib.sha256(configs.layer_weights(layer).tobytes()).digest()
            assert digest == golden[f"wsha_cfg{c}_l{li}"].tobytes(), (c, li)


def test_oracle_nan_block_fails(orc):
    blk = np.full((1, 3, 3), np.nan, dtype=complex)
    sig, fail = orc.svd_values(blk)
    assert fail[0] == 1


def test_oracle_f32_study_variant_converges(orc):
    # complex64-storage restatement used to size the fp32 tolerance floor
    layer = configs.LayerSpec(64, 64, 3, 64, 64, 2)
    w = configs.layer_weights(layer).astype(np.float64)
    fr = orc.grid_frequencies(64, 64)[[1, 100, 2000]]
    blk = orc.symbol_field(w, freqs=fr)
    ref, _ = orc.svd_values(blk)
    s, fail, sw = orc.svd_values(blk, tol=1e-6, f32="acc", return_sweeps=True)
    assert not fail.any() and sw.max() < 20
    assert per_freq_rel_err(s, ref).max() < 1e-6
