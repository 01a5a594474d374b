"""Generate the golden parity fixtures by running the REFERENCE itself.

Run in the build container (the only place /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports conv-spectra 0.1.0 read-only from /root/reference/pkg/src and
records, for seeded inputs, what the reference's own public API returns.
The output (tests/golden/golden.npz) is committed; nothing on the GPU box
reads /root/reference.

Contents (keys):
  sym_*            full symbol fields of small kernels (build_symbol_field)
  fix{i}_*         ORACLE_FIXTURES of pkg/tests/test_acceptance.py:22-28 with
                   seeds 100+i: compute_spectrum values, per-frequency sigma
                   (spectrum_from_field values_only=False), dense explicit
                   spectrum (dense_spectrum(build_explicit(..)))
  cfg{c}_l{l}_*    BASELINE configs (configs.WORKLOADS): sampled full-grid
                   frequency indices, their symbol-block Frobenius norms and
                   per-frequency singular values (descending); cfg1 complete
  blk{i}_*         svd_block triplets of seeded random complex blocks
  wsha_*           sha256 of each config's fp32 weight bytes (pins the
                   Philox generator)
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "paper_2506_05617_b200"))

import convspectra as cs  # noqa: E402  (the reference)
from convspectra.symbol import SymbolField, _symbol_blocks  # noqa: E402

import configs  # noqa: E402  (this repo's workload table; pure numpy)

ORACLE_FIXTURES = [(4, 4, 1, 1), (4, 6, 2, 3), (8, 8, 4, 2), (8, 8, 16, 16)]

# frequencies sampled per config layer (cfg1 is complete)
SAMPLES = {2: 64, 3: 32, 4: None, 5: 32}
SAMPLES_CFG4 = {64: 8, 128: 8, 256: 6, 512: 3}


def sub_field(kernel, dims, fidx):
    grid_all = cs.FrequencyGrid(dims)
    freqs = np.ascontiguousarray(grid_all.frequencies[fidx])
    grid = cs.FrequencyGrid(dims, frequencies=freqs)
    blocks = np.zeros((len(fidx), kernel.c_out, kernel.c_in), dtype=np.complex128)
    _symbol_blocks(freqs, kernel.offsets().astype(np.float64), kernel.taps(), blocks)
    return SymbolField(grid=grid, blocks=blocks)


def main():
    cs.blocksvd.resolve_workers(0)
    out = {}
    t0 = time.time()

    # symbol fields of small kernels (incl. even extents and n != m)
    for name, (co, ci, kh, kw, seed, n, m) in {
        "a": (3, 2, 3, 4, 5, 5, 3),
        "b": (2, 3, 4, 4, 21, 6, 4),
        "c": (4, 4, 3, 3, 22, 7, 5),
        "d": (2, 2, 5, 5, 23, 6, 6),
    }.items():
        k = cs.random_kernel(co, ci, kh, kw, seed=seed)
        fld = cs.build_symbol_field(k, cs.SpatialDims(n=n, m=m))
        out[f"sym_{name}_shape"] = np.array([co, ci, kh, kw, seed, n, m])
        out[f"sym_{name}_blocks"] = fld.blocks

    # acceptance oracle fixtures
    for idx, (n, m, c_in, c_out) in enumerate(ORACLE_FIXTURES):
        k = cs.random_kernel(c_out, c_in, 3, 3, seed=100 + idx)
        dims = cs.SpatialDims(n=n, m=m)
        vals = cs.compute_spectrum(k, dims).values
        _, trip = cs.spectrum_from_field(cs.build_symbol_field(k, dims), values_only=False)
        dense = cs.dense_spectrum(cs.build_explicit(k, dims, "periodic")).values
        out[f"fix{idx}_shape"] = np.array([n, m, c_in, c_out, 100 + idx])
        out[f"fix{idx}_values"] = vals
        out[f"fix{idx}_sigma"] = np.array([t.sigma for t in trip])
        out[f"fix{idx}_dense"] = dense

    # BASELINE configs
    for c, wl in configs.WORKLOADS.items():
        for li, layer in enumerate(wl.layers):
            w32 = configs.layer_weights(layer)
            out[f"wsha_cfg{c}_l{li}"] = np.frombuffer(
                hashlib.sha256(w32.tobytes()).digest(), dtype=np.uint8)
            kernel = cs.ConvKernel.from_array(w32)
            dims = cs.SpatialDims(n=layer.n, m=layer.m)
            if c == 1:
                fidx = np.arange(layer.n * layer.m)
            elif c == 4:
                if li % 4 != 0 and layer.c_out >= 256:
                    continue  # one 256/512 layer per stage keeps generation bounded
                fidx = configs.sample_frequencies(layer.n, layer.m, SAMPLES_CFG4[layer.c_out],
                                                  seed=layer.seed)
            else:
                fidx = configs.sample_frequencies(layer.n, layer.m, SAMPLES[c], seed=layer.seed)
            fld = sub_field(kernel, dims, fidx)
            res, trip = cs.spectrum_from_field(fld, values_only=False, workers=0)
            key = f"cfg{c}_l{li}"
            out[key + "_fidx"] = fidx
            out[key + "_blocknorm"] = np.linalg.norm(fld.blocks, axis=(1, 2))
            out[key + "_block0"] = fld.blocks[min(1, len(fidx) - 1)][:8, :8]
            out[key + "_sigma"] = np.array([t.sigma for t in trip])
            if c == 1:
                full = cs.compute_spectrum(kernel, dims)
                out[key + "_values"] = full.values
            print(f"{key}: {len(fidx)} freqs, {time.time() - t0:.1f}s", flush=True)

    # svd_block triplets (pkg/tests/test_blocksvd.py:15-53 shapes)
    shapes = [(3, 2), (2, 3), (4, 4), (1, 5), (6, 1), (5, 5), (16, 16), (7, 12)]
    for i, shape in enumerate(shapes):
        rng = np.random.default_rng(1000 + i)
        b = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        t = cs.svd_block(b)
        out[f"blk{i}_A"] = b
        out[f"blk{i}_U"] = t.U
        out[f"blk{i}_sigma"] = t.sigma
        out[f"blk{i}_V"] = t.V

    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB) in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
