"""Golden vectors for spectrum post-processing, from the REFERENCE itself.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_analysis.py

Runs the reference's spectral_summary / wasserstein1
(/root/reference/pkg/src/convspectra/analysis.py:35-74) on seeded spectra and
records inputs and outputs in tests/golden/golden_analysis.npz (committed;
nothing on the GPU box reads /root/reference).

Keys: sum{i}_in, sum{i}_{max,min,count,cond,mean,hist,edges};
      w1{i}_a, w1{i}_b, w1{i}_out.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import convspectra as cs  # noqa: E402  (the reference)
from convspectra.analysis import spectral_summary, wasserstein1  # noqa: E402


def spectra():
    rng = np.random.default_rng(2506)
    out = []
    # LFA spectra of the acceptance fixtures (test_acceptance.py:22-28 shapes)
    for i, (n, m, ci, co) in enumerate([(4, 4, 1, 1), (4, 6, 2, 3), (8, 8, 4, 2), (8, 8, 16, 16)]):
        k = cs.random_kernel(co, ci, 3, 3, seed=100 + i)
        out.append(cs.compute_spectrum(k, cs.SpatialDims(n, m)).values)
    out.append(np.sort(rng.uniform(0.0, 3.0, 1000))[::-1].copy())       # generic
    top = 2.75
    edges = np.linspace(0.0, top, 65)
    out.append(np.concatenate([edges, edges[::7], [top, 0.0, 0.0]]))     # values ON bin edges
    out.append(rng.integers(0, 5, 777).astype(np.float64) * 0.25)        # ties + zeros, unsorted
    out.append(np.zeros(33))                                             # smax = 0 -> top = 1
    out.append(np.array([1.5]))                                          # single value
    out.append(rng.standard_gamma(0.7, 4099) * 1e-3)                     # small, skewed, unsorted
    return out


def main():
    res = {}
    sp = spectra()
    for i, v in enumerate(sp):
        s = spectral_summary(v)
        res[f"sum{i}_in"] = v
        res[f"sum{i}_max"] = s.sigma_max
        res[f"sum{i}_min"] = s.sigma_min
        res[f"sum{i}_count"] = s.count
        res[f"sum{i}_cond"] = s.condition
        res[f"sum{i}_mean"] = s.mean
        res[f"sum{i}_hist"] = s.histogram
        res[f"sum{i}_edges"] = s.bin_edges
    pairs = [(4, 3), (3, 4), (4, 6), (9, 8), (0, 8), (3, 3), (2, 3), (5, 6), (4, 9), (1, 9)]
    for i, (a, b) in enumerate(pairs):
        res[f"w1{i}_a"] = sp[a]
        res[f"w1{i}_b"] = sp[b]
        res[f"w1{i}_out"] = wasserstein1(sp[a], sp[b])
    path = os.path.join(HERE, "golden_analysis.npz")
    np.savez_compressed(path, **res)
    print(f"wrote {path}: {len(sp)} summaries, {len(pairs)} W1 pairs")


if __name__ == "__main__":
    main()
