"""The five BASELINE.json workloads and their seeded fp32 weights.

Weights follow SURVEY.md section 8(d): the reference's Philox stream
(kernels.py:143-161, ``np.random.Generator(np.random.Philox(key=seed))``)
drawn as standard normals and He-scaled by sqrt(2/(c_in*k_h*k_w)), then cast
to float32.  Both the CUDA path and the CPU oracle consume the same fp32 bits.
Seeds: cfg1=1, cfg2=2, cfg3=3, cfg4 layer l=400+l,
cfg5=5.  The paper/reference use no public dataset, so these synthetic
weights are the whole workload.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class LayerSpec:
    c_out: int
    c_in: int
    k: int
    n: int          # torus width
    m: int          # torus height
    seed: int

    @property
    def sv_count(self) -> int:
        return self.n * self.m * min(self.c_out, self.c_in)


@dataclass(frozen=True)
class Workload:
    name: str
    layers: tuple
    vectors: bool       # singular vectors requested
    description: str

    @property
    def sv_count(self) -> int:
        return sum(layer.sv_count for layer in self.layers)


def _resnet18_stack():
    layers = []
    idx = 0
    for c, s in ((64, 56), (128, 28), (256, 14), (512, 7)):
        for _ in range(4):
            layers.append(LayerSpec(c, c, 3, s, s, 400 + idx))
            idx += 1
    return tuple(layers)


WORKLOADS = {
    1: Workload("cfg1_3x3_c16_32x32", (LayerSpec(16, 16, 3, 32, 32, 1),), False,
                "3x3 conv, c_in=c_out=16, 32x32 input, singular values"),
    2: Workload("cfg2_3x3_c64_64x64_uv", (LayerSpec(64, 64, 3, 64, 64, 2),), True,
                "3x3 conv, c=64, 64x64 input, singular values + U + V"),
    3: Workload("cfg3_3x3_256x128_56x56", (LayerSpec(256, 128, 3, 56, 56, 3),), False,
                "rectangular 3x3 conv c_in=128 c_out=256, 56x56, values only"),
    4: Workload("cfg4_resnet18_16_layers", _resnet18_stack(), False,
                "16 ResNet-18-shaped 3x3 convs, one batched call, values only"),
    5: Workload("cfg5_5x5_c256_256x256_uv", (LayerSpec(256, 256, 5, 256, 256, 5),), True,
                "5x5 conv, c=256, 256x256 input, singular values + U + V"),
}


def layer_weights(layer: LayerSpec) -> np.ndarray:
    """fp32 (c_out, c_in, k, k) He-normal weights from the Philox stream."""
    rng = np.random.Generator(np.random.Philox(key=layer.seed))
    w = rng.standard_normal((layer.c_out, layer.c_in, layer.k, layer.k))
    w = w * np.sqrt(2.0 / (layer.c_in * layer.k * layer.k))
    return w.astype(np.float32)


def sample_frequencies(n: int, m: int, count: int, seed: int = 12345) -> np.ndarray:
    """Sorted, unique full-grid indices: every self-conjugate frequency, an
    evenly spaced set, and seeded random picks (SURVEY.md 8(c) sampling)."""
    F = n * m
    picks = set()
    for i in ({0, n // 2} if n % 2 == 0 else {0}):
        for j in ({0, m // 2} if m % 2 == 0 else {0}):
            picks.add(i * m + j)
    if count >= F:
        return np.arange(F)
    for f in np.linspace(0, F - 1, max(count // 2, 1)).astype(np.int64):
        picks.add(int(f))
    rng = np.random.default_rng(seed)
    while len(picks) < count:
        picks.add(int(rng.integers(0, F)))
    return np.array(sorted(picks), dtype=np.int64)
