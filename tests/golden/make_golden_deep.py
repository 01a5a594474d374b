"""Second set of golden fixtures, made by the REFERENCE itself (round 2):
denser pins exactly where the warm-started device solver acts.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_deep.py

Imports conv-spectra 0.1.0 read-only from /root/reference/pkg/src (build
container only) and writes tests/golden/golden_deep.npz (committed; nothing
on the GPU box reads /root/reference).  Per-frequency singular values come
from the reference's own batch driver ``_svd_values_batch`` (blocksvd.py:
139-152, numba, f64, tol 1e-13) on symbol blocks from its ``_symbol_blocks``
(symbol.py:89-105) -- the same arithmetic as spectrum_from_field.

Keys:
  cfg5_deep_fidx / _sigma / _stage   >= 256 cfg5 frequencies: the 4
      self-conjugate ones, 64 at the deepest stages of the depth-8 warm plan
      (engine.warm_plan, BFS level >= 12) and seeded random representatives;
      sigma descending; the BFS stage of each frequency's representative
  cfg2_full_sigma                    every cfg2 representative (2050), the
      fp64 warm path is pinned on the full grid at 1e-10
  cfg4_l{8..15}_full_sigma           every representative of all four 256^2
      and all four 512^2 ResNet-18 layers
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import convspectra as ref  # noqa: E402  (the reference)
from convspectra.blocksvd import _svd_values_batch  # noqa: E402
from convspectra.symbol import _symbol_blocks  # noqa: E402

from paper_2506_05617_b200 import configs  # noqa: E402  (workload table)
from paper_2506_05617_b200 import engine  # noqa: E402  (host index math + warm plan, CPU)


def ref_sigma(layer, fidx):
    """Reference per-frequency sigma (descending) at full-grid indices fidx."""
    kernel = ref.ConvKernel.from_array(configs.layer_weights(layer))
    freqs = np.ascontiguousarray(ref.FrequencyGrid(ref.SpatialDims(layer.n, layer.m)).frequencies[fidx])
    blocks = np.zeros((len(fidx), kernel.c_out, kernel.c_in), dtype=np.complex128)
    _symbol_blocks(freqs, kernel.offsets().astype(np.float64), kernel.taps(), blocks)
    work = blocks if kernel.c_out >= kernel.c_in else np.ascontiguousarray(blocks.conj().transpose(0, 2, 1))
    sig, fail = _svd_values_batch(work, 1e-13, 100)
    assert not fail.any()
    return np.ascontiguousarray(sig[:, ::-1])


def main():
    ref.blocksvd.resolve_workers(0)
    out = {}
    t0 = time.time()

    # cfg5: self-conjugate + deepest warm-chain stages + random representatives
    layer = configs.WORKLOADS[5].layers[0]
    n, m = layer.n, layer.m
    total = engine.half_grid_count(n, m)
    reps = engine.half_grid_indices(n, m)
    plan = engine.warm_plan(n, m, 0, total, "cpu", engine.warm_depth(total))
    stage = np.zeros(total, dtype=np.int64)
    for d, (ids, _) in enumerate(plan):
        stage[ids.numpy()] = d
    selfc = [i * m + j for i in (0, n // 2) for j in (0, m // 2)]
    rng = np.random.default_rng(5005)
    deep = np.nonzero(stage >= 12)[0]
    deep = rng.choice(deep, size=min(64, len(deep)), replace=False)
    rand = rng.choice(total, size=192, replace=False)
    u = np.unique(np.concatenate([deep, rand, [np.searchsorted(reps, f) for f in selfc]]))
    fidx = reps[u]
    out["cfg5_deep_fidx"] = fidx
    out["cfg5_deep_stage"] = stage[u]
    out["cfg5_deep_sigma"] = ref_sigma(layer, fidx)
    print(f"cfg5: {len(fidx)} freqs (max stage {stage[u].max()}), {time.time() - t0:.1f}s", flush=True)

    # cfg2: the whole representative set
    layer = configs.WORKLOADS[2].layers[0]
    out["cfg2_full_sigma"] = ref_sigma(layer, engine.half_grid_indices(layer.n, layer.m))
    print(f"cfg2 full: {time.time() - t0:.1f}s", flush=True)

    # cfg4: all 256^2 and 512^2 layers, every representative
    for li, layer in enumerate(configs.WORKLOADS[4].layers):
        if layer.c_out < 256:
            continue
        out[f"cfg4_l{li}_full_sigma"] = ref_sigma(layer, engine.half_grid_indices(layer.n, layer.m))
        print(f"cfg4 l{li} ({layer.c_out}^2): {time.time() - t0:.1f}s", flush=True)

    path = os.path.join(HERE, "golden_deep.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
