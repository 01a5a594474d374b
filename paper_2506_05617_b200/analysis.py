"""Spectrum post-processing on the device: summaries and W1 distance.

Drop-in for the reference's ``spectral_summary`` / ``wasserstein1``
(pkg/src/convspectra/analysis.py:17-74): same names,
fields and errors, computed by the C-ABI kernels of csrc/cs_analysis.cu on the
spectrum where it already lives.  A ``SpectrumResult`` from
``compute_spectrum(..., return_device_tensors=True)`` is consumed in HBM
without a host round trip; host arrays are copied to the device first.
``boundary_compare`` (analysis.py:103-135) needs the dirichlet explicit path,
which is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, engine
from .blocksvd import SpectrumResult
from .errors import EmptySpectrum

HISTOGRAM_BINS = 64  # analysis.py:15

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


@dataclass(frozen=True)
class SpectralSummary:
    """analysis.py:18-26."""

    sigma_max: float
    sigma_min: float
    count: int
    condition: float
    mean: float
    histogram: np.ndarray = field(repr=False)
    bin_edges: np.ndarray = field(repr=False)


def _size(spectrum) -> int:
    if isinstance(spectrum, SpectrumResult):
        return len(spectrum.values)
    if torch is not None and isinstance(spectrum, torch.Tensor):
        return spectrum.numel()
    return int(np.asarray(spectrum).size)


def _device_values(spectrum, device=None):
    """The spectrum as a contiguous float64 CUDA tensor (no copy if it is one)."""
    if isinstance(spectrum, SpectrumResult):
        if spectrum.device_values is not None:
            spectrum = spectrum.device_values
        else:
            spectrum = spectrum.values
    if torch is not None and isinstance(spectrum, torch.Tensor) and spectrum.is_cuda:
        if spectrum.numel() == 0:
            raise EmptySpectrum("spectrum has no singular values")
        dev = engine.require_cuda(spectrum.device)
        return spectrum.to(torch.float64).contiguous().reshape(-1), dev
    host = np.ascontiguousarray(np.asarray(spectrum, dtype=np.float64).reshape(-1))
    if host.size == 0:  # analysis.py:40, :62 -- before any device work
        raise EmptySpectrum("spectrum has no singular values")
    dev = engine.require_cuda(device)
    return torch.from_numpy(host).to(dev), dev


def spectral_summary(spectrum, device=None) -> SpectralSummary:
    """Max / min / mean / condition plus the 64-bin histogram over [0, max]
    (analysis.py:35-53), on the device."""
    v, dev = _device_values(spectrum, device)
    n = v.numel()
    lib = _lib.load()
    stats = torch.empty(4, dtype=torch.float64, device=dev)
    counts = torch.empty(HISTOGRAM_BINS, dtype=torch.int64, device=dev)
    edges = torch.empty(HISTOGRAM_BINS + 1, dtype=torch.float64, device=dev)
    nbytes = lib.cs_analysis_workspace(n)
    ws = engine.WORKSPACE.get(dev, nbytes)
    _lib.check(lib.cs_spectral_summary(engine.ptr(v), n, engine.ptr(stats), engine.ptr(counts),
                                       engine.ptr(edges), engine.ptr(ws), nbytes,
                                       engine.stream_ptr(dev)), "spectral_summary")
    s = stats.cpu().numpy()
    smax, smin = float(s[0]), float(s[1])
    return SpectralSummary(
        sigma_max=smax,
        sigma_min=smin,
        count=int(n),
        condition=smax / smin if smin > 0 else np.inf,
        mean=float(s[2]) / n,
        histogram=counts.cpu().numpy(),
        bin_edges=edges.cpu().numpy(),
    )


def _sorted_desc(v, dev):
    lib = _lib.load()
    n = v.numel()
    out = torch.empty_like(v)
    nbytes = lib.cs_analysis_workspace(n)
    ws = engine.WORKSPACE.get(dev, nbytes)
    _lib.check(lib.cs_sort_descending_f64(engine.ptr(v), engine.ptr(out), n, engine.ptr(ws), nbytes,
                                          engine.stream_ptr(dev)), "wasserstein1 sort")
    return out


def wasserstein1(a, b, device=None) -> float:
    """W1 between two spectra via quantile coupling (analysis.py:56-74): both
    sorted descending, the shorter resampled at the longer one's quantile
    positions (np.interp semantics), mean absolute difference."""
    if _size(a) == 0 or _size(b) == 0:  # analysis.py:62-63, before any device work
        raise EmptySpectrum("wasserstein1 needs nonempty spectra")
    va, dev = _device_values(a, device)
    vb, _ = _device_values(b, dev)
    sa, sb = _sorted_desc(va, dev), _sorted_desc(vb, dev)
    lib = _lib.load()
    total = torch.empty(1, dtype=torch.float64, device=dev)
    nbytes = lib.cs_analysis_workspace(max(sa.numel(), sb.numel()))
    ws = engine.WORKSPACE.get(dev, nbytes)
    _lib.check(lib.cs_wasserstein1_sum(engine.ptr(sa), sa.numel(), engine.ptr(sb), sb.numel(),
                                       engine.ptr(total), engine.ptr(ws), nbytes,
                                       engine.stream_ptr(dev)), "wasserstein1")
    return float(total.item()) / max(sa.numel(), sb.numel())
