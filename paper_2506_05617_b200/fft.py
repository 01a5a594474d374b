"""FFT route to the symbol field (the paper's comparison baseline).

Drop-in for ``fft_symbol_field`` of pkg/src/convspectra/fft.py:103-151
(SURVEY.md 8(f) row 3): every channel pair's taps are embedded on the torus
and transformed by one batched 2D DFT (cuFFT through cs_fft_transform), and
the coefficients are gathered into per-frequency blocks (cs_fft_gather).  The
blocks agree with the LFA path to rounding; as in the reference only spectra
are contractually required to agree.  ``compute_spectrum(method="fft")``
runs this route and then the same batched SVD as the LFA path.
"""

from __future__ import annotations

import numpy as np

from . import engine
from .errors import AllocationFailure
from .kernels import ConvKernel, FrequencyGrid, SpatialDims, validate_kernel
from .symbol import (BLOCK_CONTIGUOUS, FREQUENCY_STRIDED, LAYOUTS, SymbolField, _resolve_dtype,
                     convert_layout, mem_budget_bytes)


def fft_symbol_field(kernel: ConvKernel, dims: SpatialDims, layout: str = BLOCK_CONTIGUOUS,
                     mem_budget_gib=None, *, device=None, dtype=None,
                     return_device_tensors: bool = False) -> SymbolField:
    """Per-frequency blocks via channel-pair 2D DFTs of the embedded kernel
    (fft.py:103-151).  Embedding plus transform is ``s_transform``, the gather
    into blocks ``s_copy`` (device-timed)."""
    validate_kernel(kernel)
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    dev = engine.require_cuda(device)
    dt = _resolve_dtype(kernel, dtype)
    co, ci = kernel.c_out, kernel.c_in
    esz = 8 if dt == "f32" else 16
    if return_device_tensors:
        engine.check_budget(2 * dims.size * co * ci * esz, engine.device_budget_bytes(dev, mem_budget_gib),
                            f"fft field ({co * ci} embedded {dims.m}x{dims.n} grids + blocks)")
    else:
        need = 2 * dims.size * co * ci * 16  # fft.py:123-130
        budget = mem_budget_bytes(mem_budget_gib)
        if need > budget:
            raise AllocationFailure(
                f"fft path needs {need} bytes for {co * ci} embedded {dims.m}x{dims.n} grids "
                f"plus the block field, budget is {budget} bytes")
    w = engine.weights_to_device(kernel, dt, dev)
    tm = engine.Timer(dev)
    tm.mark("t0")
    full = engine.fft_symbol_field(w, dims.n, dims.m, dt, half=False, timer=tm)
    tm.mark("t1")
    blocks = full if return_device_tensors else full.cpu().numpy().astype(np.complex128)
    fld = SymbolField(grid=FrequencyGrid(dims), blocks=blocks, layout=BLOCK_CONTIGUOUS, source="fft",
                      s_transform=tm.seconds("t0", "tf"), s_copy=tm.seconds("tf", "t1"), dtype=dt)
    if layout == FREQUENCY_STRIDED:
        fld = convert_layout(fld, FREQUENCY_STRIDED)
    return fld
