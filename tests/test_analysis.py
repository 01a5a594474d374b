"""Spectrum post-processing: the device
spectral_summary / wasserstein1 (csrc/cs_analysis.cu) against goldens recorded
from the reference's analysis.py:35-74 (tests/golden/make_golden_analysis.py),
and the oracle restatement pinned to the same goldens."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402

GOLD = np.load(os.path.join(ROOT, "tests", "golden", "golden_analysis.npz"))
NSUM = len([k for k in GOLD.files if k.endswith("_hist")])
NW1 = len([k for k in GOLD.files if k.endswith("_out")])


@pytest.mark.parametrize("i", range(NSUM))
def test_oracle_summary_pinned(i):
    hi, lo, cnt, cond, mean, hist, edges = orc.summary(GOLD[f"sum{i}_in"])
    assert hi == GOLD[f"sum{i}_max"] and lo == GOLD[f"sum{i}_min"] and cnt == GOLD[f"sum{i}_count"]
    assert cond == GOLD[f"sum{i}_cond"] and mean == GOLD[f"sum{i}_mean"]
    assert np.array_equal(hist, GOLD[f"sum{i}_hist"]) and np.array_equal(edges, GOLD[f"sum{i}_edges"])


@pytest.mark.parametrize("i", range(NW1))
def test_oracle_w1_pinned(i):
    assert orc.w1(GOLD[f"w1{i}_a"], GOLD[f"w1{i}_b"]) == GOLD[f"w1{i}_out"]


def test_empty_spectrum_raises_before_device_work():
    import paper_2506_05617_b200 as cs
    with pytest.raises(cs.EmptySpectrum):
        cs.spectral_summary(np.zeros(0))
    with pytest.raises(cs.EmptySpectrum):
        cs.wasserstein1([1.0, 2.0], [])


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(NSUM))
def test_device_summary_matches_reference(cuda, i):
    import paper_2506_05617_b200 as cs
    s = cs.spectral_summary(GOLD[f"sum{i}_in"])
    assert s.sigma_max == GOLD[f"sum{i}_max"] and s.sigma_min == GOLD[f"sum{i}_min"]
    assert s.count == GOLD[f"sum{i}_count"] and s.condition == GOLD[f"sum{i}_cond"]
    # fp64 sums in another order than numpy's pairwise sum: a few ulp
    assert abs(s.mean - GOLD[f"sum{i}_mean"]) <= 1e-13 * max(abs(GOLD[f"sum{i}_mean"]), 1e-300)
    assert np.array_equal(s.histogram, GOLD[f"sum{i}_hist"])  # integer counts: exact
    assert np.array_equal(s.bin_edges, GOLD[f"sum{i}_edges"])


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(NW1))
def test_device_w1_matches_reference(cuda, i):
    import paper_2506_05617_b200 as cs
    ref = float(GOLD[f"w1{i}_out"])
    got = cs.wasserstein1(GOLD[f"w1{i}_a"], GOLD[f"w1{i}_b"])
    assert abs(got - ref) <= 1e-13 * max(ref, 1e-300) + 1e-300


@pytest.mark.gpu
def test_device_analysis_on_device_spectrum(cuda):
    """cfg2 spectrum kept in HBM: summary and W1 against the oracle on its
    host copy; Parseval-style invariants of the summary."""
    import torch
    import paper_2506_05617_b200 as cs
    from paper_2506_05617_b200 import configs
    from paper_2506_05617_b200.pipeline import lfa_device
    layer = configs.WORKLOADS[2].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(cuda)
    res = lfa_device(w, layer.n, layer.m, "f32", False)
    vals = res.values
    host = vals.cpu().numpy()
    s = cs.spectral_summary(vals)
    hi, lo, cnt, cond, mean, hist, edges = orc.summary(host)
    assert (s.sigma_max, s.sigma_min, s.count) == (hi, lo, cnt)
    assert np.array_equal(s.histogram, hist) and np.array_equal(s.bin_edges, edges)
    assert abs(s.mean - mean) <= 1e-12 * mean
    half = host[::2].copy()
    assert abs(cs.wasserstein1(vals, half) - orc.w1(host, half)) <= 1e-12 * orc.w1(host, half)
    with pytest.raises(cs.EmptySpectrum):
        cs.wasserstein1(vals, np.zeros(0))
