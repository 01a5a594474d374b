"""Batched complex SVD of symbol blocks and spectrum assembly (drop-in for
pkg/src/convspectra/blocksvd.py), computed by the library's sm_100a kernels.

Result types and their invariants are the reference's (blocksvd.py:29-66,
SPEC.md:51-62): values descending, length F*min(c_in,c_out), U^H U = I,
V^H V = I, A_f = U diag(sigma) V^H.  ``workers`` is accepted for signature
compatibility; results never depend on it (the reference guarantees the
same bit-for-bit across worker counts).
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import engine
from .engine import DEFAULT_MAX_SWEEPS, DEFAULT_SVD_TOL
from .errors import IndexOutOfRange
from .kernels import SpatialDims


@dataclass(frozen=True)
class PhaseTimings:
    """Device-timed split of a spectrum computation (CUDA events)."""

    s_transform: float
    s_svd: float
    s_copy: float
    s_total: float

    @classmethod
    def build(cls, s_transform, s_svd, s_copy=0.0):
        return cls(s_transform=s_transform, s_svd=s_svd, s_copy=s_copy,
                   s_total=s_transform + s_svd + s_copy)


@dataclass(frozen=True)
class SvdTriplet:
    """Per-frequency factors A_k = U diag(sigma) V^*."""

    k: Optional[tuple]
    U: object
    sigma: object
    V: object


@dataclass(frozen=True)
class SpectrumResult:
    """Descending singular values plus provenance metadata.

    ``device_values`` optionally holds the same values as a CUDA tensor."""

    values: np.ndarray = field(repr=False)
    method: str
    boundary: str
    dims: SpatialDims
    channels: tuple
    timings: Optional[PhaseTimings] = None
    device_values: object = field(default=None, repr=False, compare=False)

    def __len__(self):
        return len(self.values)


def sort_descending(values: np.ndarray) -> np.ndarray:
    """Stable descending sort of host values; ties keep input order (blocksvd.py:69-72)."""
    values = np.asarray(values)
    return values[np.argsort(-values, kind="stable")]


def resolve_workers(workers) -> int:
    """Kept for API compatibility: the device path has no host thread pool."""
    if not workers:
        return os.cpu_count() or 1
    return max(1, int(workers))


def _to_device_blocks(blocks, dev, dtype):
    torch = engine.torch
    want = engine.complex_dtype(dtype)
    if isinstance(blocks, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(blocks)).to(dev)
    else:
        t = blocks.to(dev)
    if t.dtype != want:
        t = t.to(want)
    return t.contiguous()


def _infer_dtype(fld_or_blocks, dtype):
    if dtype is not None:
        return "f32" if dtype in ("f32", "float32", "complex64") else "f64"
    b = getattr(fld_or_blocks, "blocks", fld_or_blocks)
    dt = getattr(fld_or_blocks, "dtype", None)
    if isinstance(dt, str) and dt in ("f32", "f64"):
        return dt
    return "f32" if str(b.dtype) in ("complex64", "torch.complex64") else "f64"


def svd_block(block, k=None, tol=DEFAULT_SVD_TOL, max_sweeps=DEFAULT_MAX_SWEEPS, *,
              device=None, dtype=None) -> SvdTriplet:
    """Full SVD of one c_out x c_in complex block (blocksvd.py:227-237)."""
    b = np.atleast_2d(np.asarray(block, dtype=np.complex128))
    dev = engine.require_cuda(device)
    dt = "f64" if dtype is None else _infer_dtype(b, dtype)
    engine.check_tol(tol, dt, max(b.shape))
    t = _to_device_blocks(b[None], dev, dt)
    out = engine.batched_svd(t, dt, True, tol, max_sweeps)
    f = engine.first_failure(out.info)
    if f >= 0:
        engine.raise_convergence(f, None, max_sweeps)
    return SvdTriplet(k=k, U=out.U[0].cpu().numpy().astype(np.complex128),
                      sigma=out.sigma[0].cpu().numpy().astype(np.float64),
                      V=out.V[0].cpu().numpy().astype(np.complex128))


def spectrum_from_field(fld, values_only: bool = True, workers: int = 1,
                        tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS, *,
                        device=None, dtype=None, return_device_tensors: bool = False):
    """SVD every block of a symbol field and merge the singular values
    (blocksvd.py:240-289).

    A full-grid field that is exactly conjugate-symmetric (every field this
    package builds) is solved on its conjugate-orbit representatives only;
    any other field (caller-modified, sub-grid) is solved block by block, so
    failures are reported at the reference's frequency index."""
    resolve_workers(workers)
    torch = engine.torch
    blocks = fld.blocks
    dev = engine.require_cuda(device if device is not None else
                              (blocks.device if hasattr(blocks, "device") and
                               getattr(blocks.device, "type", "") == "cuda" else None))
    dt = _infer_dtype(fld, dtype)
    F, co, ci = blocks.shape
    grid = fld.grid
    n, m = grid.dims.n, grid.dims.m
    tm = engine.Timer(dev)
    t = _to_device_blocks(blocks, dev, dt)
    full_grid = F == n * m and len(grid.frequencies) == n * m
    half = full_grid and engine.is_conj_symmetric(t, n, m, dt)
    reps = engine.half_grid_indices(n, m) if half else None

    engine.check_tol(tol, dt, max(co, ci))
    tm.mark("t0")
    work = t.index_select(0, torch.from_numpy(reps).to(dev)) if half else t
    # values_only=True runs the vectors solve when that is the panel kernel, so
    # values agree bitwise with values_only=False (blocksvd.py:4-8, T/test_blocksvd.py:110-116)
    vec = (not values_only) or engine.values_via_vectors(work.shape[0], co, ci, dt)
    out = engine.batched_svd(work, dt, vec, tol, max_sweeps)
    values_dev = engine.spectrum_values(out.sigma, dt, n, m, half)
    ffail = engine.first_failure(out.info)
    tm.mark("t1")
    if ffail >= 0:
        fidx = int(reps[ffail]) if half else ffail
        engine.raise_convergence(fidx, grid.frequencies, max_sweeps)
    s_svd = tm.seconds("t0", "t1")
    values = values_dev.cpu().numpy()
    result = SpectrumResult(values=values, method=fld.source, boundary="periodic",
                            dims=grid.dims, channels=(ci, co),
                            timings=engine_timings(fld, s_svd),
                            device_values=values_dev if return_device_tensors else None)
    if values_only:
        return result
    trip = TripletList(out.sigma, out.U, out.V, grid.frequencies, n, m, half,
                       host=not return_device_tensors)
    return result, trip


class TripletList:
    """Per-frequency triplets in grid order, materialised on access.

    The reference returns a list whose U/V are views into shared batch
    arrays (blocksvd.py:271-275).  Here the factors stay on the device at
    their solved size: for a conjugate-symmetric field only the
    representatives are stored and the partner f* of a representative u gets
    U_f* = conj(U_u), V_f* = conj(V_u), sigma_f* = sigma_u -- the
    full cfg5 grid (2 x 34 GB of fp32 factors expanded, 2 x 69 GB as host
    complex128) is never built.  Item access returns an SvdTriplet with host
    complex128 / float64 arrays (host=True, the reference's types) or device
    tensors; indexing, iteration, len() and slices work like the list."""

    def __init__(self, sigma, U, V, freqs, n, m, half, host=True):
        self._sig, self._U, self._V = sigma, U, V
        self._freqs = freqs
        self._host = host
        self._n = len(freqs)
        if half:
            rep_of, conj = engine.partner_map(n, m)
            self._rep, self._conj = rep_of, conj
        else:
            self._rep, self._conj = np.arange(self._n), np.zeros(self._n, dtype=bool)

    def __len__(self):
        return self._n

    def __iter__(self):
        for f in range(self._n):
            yield self[f]

    def __getitem__(self, f):
        if isinstance(f, slice):
            return [self[i] for i in range(*f.indices(self._n))]
        f = int(f)
        if f < 0:
            f += self._n
        if not 0 <= f < self._n:
            raise IndexError(f"frequency index {f} out of range for {self._n} frequencies")
        u, cj = int(self._rep[f]), bool(self._conj[f])
        Uf, Vf, sf = self._U[u], self._V[u], self._sig[u]
        if cj:  # materialised copies: a lazy torch conj view would reach the C-ABI unconjugated
            Uf, Vf = Uf.conj().resolve_conj(), Vf.conj().resolve_conj()
        if self._host:
            Uf = Uf.cpu().numpy().astype(np.complex128)
            Vf = Vf.cpu().numpy().astype(np.complex128)
            sf = sf.cpu().numpy().astype(np.float64)
        k = (self._freqs[f, 0], self._freqs[f, 1])
        return SvdTriplet(k=k, U=Uf, sigma=sf, V=Vf)


def engine_timings(fld, s_svd: float) -> PhaseTimings:
    return PhaseTimings.build(getattr(fld, "s_transform", 0.0), s_svd, getattr(fld, "s_copy", 0.0))


def materialize_singular_vector(triplet: SvdTriplet, column: int, side: str,
                                dims: SpatialDims) -> np.ndarray:
    """Global spatial singular vector of one frequency / factor column
    (blocksvd.py:292-311): entry (x1*n + x2)*c + ch equals
    exp(2 pi i (k1 x2 + k2 x1)) / sqrt(nm) * W[ch, column]."""
    if side not in ("left", "right"):
        raise ValueError(f"side must be 'left' or 'right', got {side!r}")
    W = triplet.U if side == "left" else triplet.V
    if not 0 <= column < W.shape[1]:
        raise IndexOutOfRange(f"column {column} out of range for rank {W.shape[1]}")
    n, m = dims.n, dims.m
    k1, k2 = triplet.k
    if not isinstance(W, np.ndarray):
        # device factors: the vector is formed on the device (cs_materialize_vector)
        fi, fj = int(round(float(k1) * n)) % n, int(round(float(k2) * m)) % m
        if abs(fi - float(k1) * n) > 1e-9 * n or abs(fj - float(k2) * m) > 1e-9 * m:
            raise ValueError("device materialisation needs a grid frequency")
        dt = "f32" if W.dtype == engine.torch.complex64 else "f64"
        return engine.materialize_vector(W, column, fi, fj, n, m, dt)
    x1, x2 = np.divmod(np.arange(n * m), n)
    wave = np.exp(2j * np.pi * (k1 * x2 + k2 * x1)) / np.sqrt(n * m)
    return (wave[:, None] * np.asarray(W)[None, :, column]).ravel()
