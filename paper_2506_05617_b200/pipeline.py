"""End-to-end spectrum computation: the drop-in ``compute_spectrum``.

The reference dispatches on ``method`` at pkg/src/convspectra/pipeline.py:
52-68; the "lfa" branch (build_symbol_field -> spectrum_from_field) is the
hot path this package replaces.  The B200 path never materialises the full
field: K1 assembles the conjugate-orbit representatives straight into HBM,
the batched Jacobi solves them in place, and the spectrum assembly emits
every value twice for non-self-conjugate representatives before one device
sort.  With ``values_only=False`` the factors are computed and discarded,
exactly as the reference does (pipeline.py:37-43, 69); use
``spectrum_from_field`` or :func:`lfa_device` to keep them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import engine
from .blocksvd import PhaseTimings, SpectrumResult, resolve_workers
from .engine import DEFAULT_MAX_SWEEPS, DEFAULT_SVD_TOL
from .kernels import ConvKernel, SpatialDims, validate_kernel
from .symbol import BLOCK_CONTIGUOUS, LAYOUTS, _resolve_dtype

METHODS = ("lfa", "fft", "explicit")
PERIODIC = "periodic"
DIRICHLET = "dirichlet"
BOUNDARIES = (PERIODIC, DIRICHLET)


@dataclass
class DeviceSpectrum:
    """Device-resident outputs of one LFA solve over representatives [u0, u0+count)."""

    values: object          # float64 (n*m*r,) descending, or None when sharded
    sigma: object           # (count, r) per representative, descending
    U: object               # (count, c_out, r) or None
    V: object               # (count, c_in, r) or None
    info: object            # (count,) int32 sweeps or -1
    u0: int
    count: int
    dtype: str
    ids: object = None      # representative indices of the rows (shards), or None: u0 + arange


def lfa_device(w_dev, n: int, m: int, dtype: str, want_vectors: bool = False,
               tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS,
               u0: int = 0, count: int | None = None, assemble: bool = True,
               timer: engine.Timer | None = None, field_out=None,
               warm_start=None, method: str = "lfa", ids=None) -> DeviceSpectrum:
    """K1 -> K2/K3 -> assembly on the current stream, no host synchronisation.

    Solves the representatives [u0, u0+count), or the representative set
    ``ids`` (sorted; whole warm-start trees, distributed.shard_ids) -- then
    every block is solved exactly as in the whole-grid solve, so shards
    reproduce it bit for bit.  ``warm_start`` (default: when vectors are
    requested and the panel kernel applies) solves each block of the
    warm-start forest from its solved lattice neighbour's right factor."""
    total = engine.half_grid_count(n, m)
    if ids is not None:
        ids = np.asarray(ids, dtype=np.int64)
        u0, count = int(ids[0]), len(ids)
    elif count is None:
        count = total - u0
    if timer:
        timer.mark("t0")
    if method == "fft":  # fft.py route to the same representative blocks
        if u0 != 0 or count != total:
            raise ValueError("the FFT route builds the whole half grid (u0=0, count=None)")
        fld = engine.fft_symbol_field(w_dev, n, m, dtype, half=True, timer=timer, out=field_out)
    elif ids is not None:  # K1 over the covering range, then the shard's blocks
        span = int(ids[-1]) - u0 + 1
        rng = engine.symbol_field(w_dev, n, m, dtype, half=True, f_first=u0, f_count=span)
        fld = rng if span == count else rng.index_select(0, torch_ids(ids - u0, w_dev.device))
        del rng
    else:
        fld = engine.symbol_field(w_dev, n, m, dtype, half=True, f_first=u0, f_count=count,
                                  out=field_out)
    if timer:
        timer.mark("t1")
    co, ci = w_dev.shape[0], w_dev.shape[1]
    decide = total if ids is not None else count  # shards decide as the whole grid does
    if (engine.use_warm_start(decide, co, ci, dtype, want_vectors, warm_start) or
            (not want_vectors and warm_start is None and engine.use_warm_values(decide, co, ci, dtype))):
        out = engine.batched_svd_warm(fld, dtype, n, m, u0, tol, max_sweeps, ids=ids)
        if not want_vectors:
            out.U = out.V = None
    elif ids is not None:  # cold, planned as the whole grid
        out = engine.alloc_svd_outputs(count, co, ci, dtype, want_vectors, fld.device)
        engine.batched_svd_indexed(fld, dtype, want_vectors, None, out, tol, max_sweeps,
                                   plan_count=total)
        if want_vectors:
            engine.complete_zero_columns(out, co, ci, dtype)
    else:
        out = engine.batched_svd(fld, dtype, want_vectors, tol, max_sweeps)
    if timer:
        timer.mark("t2")
    values = None
    if assemble and u0 == 0 and count == total:
        values = engine.spectrum_values(out.sigma, dtype, n, m, True)
    if timer:
        timer.mark("t3")
    return DeviceSpectrum(values, out.sigma, out.U, out.V, out.info, u0, count, dtype, ids)


def torch_ids(ids, device):
    return engine.torch.from_numpy(np.ascontiguousarray(ids, dtype=np.int64)).to(device)


def lfa_device_multi(layers, dtype: str, want_vectors: bool = False,
                     tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS,
                     timer: engine.Timer | None = None):
    """Several layers in ONE batched SVD call (cfg4: 16 ResNet-18 layers).

    ``layers`` = [(w_dev, n, m), ...].  K1 runs per layer, then a single
    cs_batched_svd_grouped call solves every layer's representatives with
    its own kernel configuration, the groups running concurrently on forked
    streams so small and large shapes share the SMs."""
    if timer:
        timer.mark("t0")
    fields = [engine.symbol_field(w, n, m, dtype, half=True) for w, n, m in layers]
    if timer:
        timer.mark("t1")
    # layers of one block shape share one group (one fuller launch instead of
    # several partial waves: cfg4's four 512^2 layers are 4 x 25 blocks)
    by_shape = {}
    for i, f in enumerate(fields):
        by_shape.setdefault(tuple(f.shape[1:]), []).append(i)
    merged = [fields[ix[0]] if len(ix) == 1 else engine.torch.cat([fields[i] for i in ix])
              for ix in by_shape.values()]
    mouts = engine.batched_svd_grouped(merged, dtype, want_vectors, tol, max_sweeps)
    outs = [None] * len(fields)
    for ix, mo in zip(by_shape.values(), mouts):
        off = 0
        for i in ix:
            c = fields[i].shape[0]
            cut = (lambda t: None if t is None else t[off:off + c])  # noqa: E731
            outs[i] = engine.SvdBatch(sigma=mo.sigma[off:off + c], info=mo.info[off:off + c],
                                      U=cut(mo.U), V=cut(mo.V), zero=cut(mo.zero))
            off += c
    if timer:
        timer.mark("t2")
    res = []
    for (w, n, m), o in zip(layers, outs):
        vals = engine.spectrum_values(o.sigma, dtype, n, m, True)
        res.append(DeviceSpectrum(vals, o.sigma, o.U, o.V, o.info, 0, o.sigma.shape[0], dtype))
    if timer:
        timer.mark("t3")
    return res


def compute_spectra(kernels, dims, values_only: bool = True, tol: float = DEFAULT_SVD_TOL,
                    max_sweeps: int = DEFAULT_MAX_SWEEPS, *, device=None, dtype=None):
    """``compute_spectrum`` for a list of layers in one batched device call
    (extension: the reference solves one kernel per call).  ``dims`` is one
    SpatialDims or one per kernel.  Returns a list of SpectrumResult."""
    from .kernels import FrequencyGrid

    kernels = list(kernels)
    dims_l = list(dims) if isinstance(dims, (list, tuple)) else [dims] * len(kernels)
    dev = engine.require_cuda(device)
    dt = _resolve_dtype(kernels[0] if kernels else None, dtype)
    for k in kernels:
        validate_kernel(k)
    for k in kernels:
        engine.check_tol(tol, dt, max(k.c_out, k.c_in))
    layers = [(engine.weights_to_device(k, dt, dev), d.n, d.m) for k, d in zip(kernels, dims_l)]
    tm = engine.Timer(dev)
    outs = lfa_device_multi(layers, dt, not values_only, tol, max_sweeps, timer=tm)
    results = []
    for k, d, o in zip(kernels, dims_l, outs):
        f = engine.first_failure(o.info)
        if f >= 0:
            reps = engine.half_grid_indices(d.n, d.m)
            engine.raise_convergence(int(reps[f]), FrequencyGrid(d).frequencies, max_sweeps)
    timings = PhaseTimings.build(tm.seconds("t0", "t1"), tm.seconds("t1", "t3"), 0.0)
    for k, d, o in zip(kernels, dims_l, outs):
        results.append(SpectrumResult(values=o.values.cpu().numpy(), method="lfa",
                                      boundary=PERIODIC, dims=d, channels=(k.c_in, k.c_out),
                                      timings=timings))
    return results


def field_bytes(kernel_or_shape, n: int, m: int, dtype: str, want_vectors: bool) -> int:
    co, ci = kernel_or_shape
    esz = 8 if dtype == "f32" else 16
    F_u = engine.half_grid_count(n, m)
    r = min(co, ci)
    need = F_u * co * ci * esz
    if want_vectors:
        need += F_u * (co + ci) * r * esz
    return need


def compute_spectrum(kernel: ConvKernel, dims: SpatialDims, method: str = "lfa",
                     boundary: str = PERIODIC, values_only: bool = True, workers: int = 0,
                     layout: str = BLOCK_CONTIGUOUS, size_cap=None, mem_budget_gib=None,
                     tol: float = DEFAULT_SVD_TOL, max_sweeps: int = DEFAULT_MAX_SWEEPS, *,
                     device=None, dtype=None,
                     return_device_tensors: bool = False) -> SpectrumResult:
    """Full singular value spectrum with device phase timings attached
    (pipeline.py:24-69).  Only the LFA method is on this package's hot path;
    "fft" and "explicit" are the reference's comparison/oracle routes."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    if boundary not in BOUNDARIES:
        raise ValueError(f"unknown boundary {boundary!r}")
    if boundary == DIRICHLET and method != "explicit":
        raise ValueError(f"method {method!r} only supports periodic boundaries")
    if method == "explicit":
        raise NotImplementedError(
            "method 'explicit' (the dense oracle, explicit.py) is outside the B200 hot path")
    if layout not in LAYOUTS:
        raise ValueError(f"unknown layout {layout!r}")
    resolve_workers(workers)
    validate_kernel(kernel)
    dev = engine.require_cuda(device)
    dt = _resolve_dtype(kernel, dtype)
    n, m = dims.n, dims.m
    co, ci = kernel.c_out, kernel.c_in
    engine.check_tol(tol, dt, max(co, ci))
    # values_only=True runs the same solve as values_only=False whenever that
    # solve is the panel / tensor-core kernel, so the two return bitwise equal
    # values (the reference's guarantee, pipeline.py:40-42); the factors are
    # computed and dropped
    vec = (not values_only) or engine.values_via_vectors(engine.half_grid_count(n, m), co, ci, dt)
    need = field_bytes((co, ci), n, m, dt, vec)
    if method == "fft":  # plus the embedded channel-pair grids (fft.py:123-130)
        need += co * ci * n * m * (8 if dt == "f32" else 16)
    engine.check_budget(need, engine.device_budget_bytes(dev, mem_budget_gib),
                        f"{method.upper()} solve ({engine.half_grid_count(n, m)} blocks of {co}x{ci})")
    w = engine.weights_to_device(kernel, dt, dev)
    tm = engine.Timer(dev)
    res = lfa_device(w, n, m, dt, vec, tol, max_sweeps, timer=tm, method=method)
    res.U = res.V = None  # compute_spectrum returns values only (pipeline.py:69)
    f = engine.first_failure(res.info)
    if f >= 0:
        reps = engine.half_grid_indices(n, m)
        from .kernels import FrequencyGrid
        engine.raise_convergence(int(reps[f]), FrequencyGrid(dims).frequencies, max_sweeps)
    if method == "fft":  # s_transform = embed + DFT, s_copy = gather (fft.py:139-146)
        timings = PhaseTimings.build(tm.seconds("t0", "tf"), tm.seconds("t1", "t3"),
                                     tm.seconds("tf", "t1"))
    else:
        timings = PhaseTimings.build(tm.seconds("t0", "t1"), tm.seconds("t1", "t3"), 0.0)
    values = res.values.cpu().numpy()
    return SpectrumResult(values=values, method=method, boundary=PERIODIC, dims=dims,
                          channels=(ci, co), timings=timings,
                          device_values=res.values if return_device_tensors else None)
