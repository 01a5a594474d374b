"""Symbol fields: one c_out x c_in complex block per torus frequency.

Drop-in for pkg/src/convspectra/symbol.py.  The blocks are computed on the
B200 by K1 (cs_symbol_field): only the conjugate-orbit representatives are
assembled, and the full grid is their conj() mirror (cs_expand_half_grid),
so the field is exactly conjugate-symmetric.  By default ``blocks`` is a
host numpy complex128 array (the reference's type, and the reference's
16 GiB budget applies to it); ``return_device_tensors=True`` keeps the field
on the device as a torch tensor in the compute precision.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field

import numpy as np

from . import engine
from .errors import AllocationFailure
from .kernels import ConvKernel, FrequencyGrid, SpatialDims, validate_kernel

BLOCK_CONTIGUOUS = "block_contiguous"
FREQUENCY_STRIDED = "frequency_strided"
LAYOUTS = (BLOCK_CONTIGUOUS, FREQUENCY_STRIDED)

DEFAULT_MEM_BUDGET_GIB = 16.0
MEM_BUDGET_ENV = "CONV_SPECTRA_MEM_BUDGET_GIB"


def mem_budget_bytes(mem_budget_gib=None) -> int:
    """Host field budget: parameter, then env, then 16 GiB (symbol.py:27-35)."""
    if mem_budget_gib is None:
        mem_budget_gib = float(os.environ.get(MEM_BUDGET_ENV, DEFAULT_MEM_BUDGET_GIB))
    return int(float(mem_budget_gib) * 2**30)


@dataclass(frozen=True)
class SymbolField:
    """Blocks (F, c_out, c_in) over a frequency grid plus a layout tag.

    ``blocks`` is numpy (host) or a torch CUDA tensor (device).  ``dtype`` is
    the precision the blocks were computed in ("f32"/"f64")."""

    grid: FrequencyGrid
    blocks: object = field(repr=False)
    layout: str = BLOCK_CONTIGUOUS
    source: str = "lfa"
    s_transform: float = 0.0
    s_copy: float = 0.0
    dtype: str = "f64"

    @property
    def c_out(self) -> int:
        return int(self.blocks.shape[1])

    @property
    def c_in(self) -> int:
        return int(self.blocks.shape[2])

    def block(self, f: int):
        return self.blocks[f]


def _resolve_dtype(kernel: ConvKernel, dtype) -> str:
    """Compute precision.  The reference computes in float64 whatever the
    weights' precision tag (kernels.py:40, symbol.py:134), so the drop-in does
    too; fp32 (the measured complex64 mode, 1e-5 of sigma_max per frequency)
    is an explicit opt-in with dtype="f32"."""
    if dtype is None:
        return "f64"
    if dtype in ("f32", "float32", "complex64"):
        return "f32"
    if dtype in ("f64", "float64", "complex128"):
        return "f64"
    raise ValueError(f"unknown dtype {dtype!r}")


def symbol_at(kernel: ConvKernel, k, *, device=None, dtype=None) -> np.ndarray:
    """Symbol block at one frequency pair k (symbol.py:74-86), on the device."""
    validate_kernel(kernel)
    dev = engine.require_cuda(device)
    dt = _resolve_dtype(kernel, dtype)
    w = engine.weights_to_device(kernel, dt, dev)
    out = engine.symbol_at_freqs(w, np.asarray([k], dtype=np.float64), dt)
    return out[0].cpu().numpy().astype(np.complex128)


def build_symbol_field(kernel: ConvKernel, dims: SpatialDims, layout: str = BLOCK_CONTIGUOUS,
                       mem_budget_gib=None, *, device=None, dtype=None,
                       return_device_tensors: bool = False) -> SymbolField:
    """Evaluate the symbol on the full frequency grid (symbol.py:108-143).

    Raises AllocationFailure before allocating when the complex128 host field
    would exceed the budget (same rule as the reference); device-resident
    fields are checked against the device budget instead."""
    validate_kernel(kernel)
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    dev = engine.require_cuda(device)
    dt = _resolve_dtype(kernel, dtype)
    F = dims.size
    co, ci = kernel.c_out, kernel.c_in
    if return_device_tensors:
        esz = 8 if dt == "f32" else 16
        engine.check_budget(F * co * ci * esz, engine.device_budget_bytes(dev, mem_budget_gib),
                            f"symbol field ({F} blocks of {co}x{ci})")
    else:
        need = F * co * ci * 16
        budget = mem_budget_bytes(mem_budget_gib)
        if need > budget:
            raise AllocationFailure(
                f"symbol field needs {need} bytes ({F} blocks of {co}x{ci} complex128), "
                f"budget is {budget} bytes")
    grid = FrequencyGrid(dims)
    w = engine.weights_to_device(kernel, dt, dev)
    tm = engine.Timer(dev)
    tm.mark("t0")
    half = engine.symbol_field(w, dims.n, dims.m, dt, half=True)
    full = engine.expand_half(half, dims.n, dims.m, dt)
    del half
    tm.mark("t1")
    s_transform = tm.seconds("t0", "t1")
    blocks = full if return_device_tensors else full.cpu().numpy().astype(np.complex128)
    fld = SymbolField(grid=grid, blocks=blocks, layout=BLOCK_CONTIGUOUS,
                      s_transform=s_transform, dtype=dt)
    if layout == FREQUENCY_STRIDED:
        fld = convert_layout(fld, FREQUENCY_STRIDED)
    return fld


def convert_layout(fld: SymbolField, layout: str) -> SymbolField:
    """Re-store the blocks; values are bit-identical (symbol.py:146-161)."""
    import time

    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    if layout == fld.layout:
        return fld
    t0 = time.perf_counter()
    b = fld.blocks
    is_np = isinstance(b, np.ndarray)
    if layout == FREQUENCY_STRIDED:
        base = np.ascontiguousarray(b.transpose(1, 2, 0)) if is_np else b.permute(1, 2, 0).contiguous()
        blocks = base.transpose(2, 0, 1) if is_np else base.permute(2, 0, 1)
    else:
        blocks = np.ascontiguousarray(b) if is_np else b.contiguous()
    if not is_np:
        engine.torch.cuda.synchronize(blocks.device)
    s_copy = time.perf_counter() - t0
    return SymbolField(grid=fld.grid, blocks=blocks, layout=layout, source=fld.source,
                       s_transform=fld.s_transform, s_copy=fld.s_copy + s_copy, dtype=fld.dtype)
