"""ctypes front-end of the CPU oracle (oracle.c).

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  The product package
(paper_2506_05617_b200) never imports this module.

Restates the reference's host-side glue around the numba kernels:

* ``grid_frequencies``   <- kernels.py:126-134 (k = (i/n, j/m), row-major f=i*m+j)
* ``offsets`` / ``taps`` <- kernels.py:63-68, 71-85
* ``symbol_field``       <- symbol.py:108-137 (np.zeros + _symbol_blocks)
* ``svd_values``         <- blocksvd.py:253-264 (wide -> conj transpose,
                            _svd_values_batch, sig[:, ::-1])
* ``svd_full``           <- blocksvd.py:184-210, 266-270 (_finish_full,
                            _complete_zero_columns, U/V swap for wide blocks)
* ``spectrum_values``    <- pipeline.py:61-69 + blocksvd.py:276 (global
                            stable descending sort)
* ``summary``            <- analysis.py:35-53 (max/min/mean/condition, 64-bin
                            histogram over [0, top])
* ``w1``                 <- analysis.py:56-74 (quantile-coupled W1)
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

DEFAULT_TOL = 1e-13        # blocksvd.py:26
DEFAULT_MAX_SWEEPS = 100   # blocksvd.py:25

_dp = ctypes.POINTER(ctypes.c_double)
_fp = ctypes.POINTER(ctypes.c_float)
_i8p = ctypes.POINTER(ctypes.c_int8)
_i32p = ctypes.POINTER(ctypes.c_int32)


def build():
    """Compile liboracle.so in place (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = ctypes.CDLL(path)
        L.orc_symbol_blocks.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int, _dp,
                                        ctypes.c_int, ctypes.c_int, _dp, ctypes.c_int]
        for name, p in (("orc_svd_values_batch", _dp), ("orc_svd_values_batch_f32", _fp),
                        ("orc_svd_values_batch_f32acc", _fp)):
            getattr(L, name).argtypes = [p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_int, _dp, _i8p, _i32p,
                                         ctypes.c_int]
        L.orc_svd_full_batch.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_int, _dp, _dp, _dp,
                                         _i8p, _i32p, ctypes.c_int]
        L.orc_max_threads.restype = ctypes.c_int
        _LIB = L
    return _LIB


def max_threads() -> int:
    return int(lib().orc_max_threads())


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t)


# kernels.py:71-85
def offsets(k_h: int, k_w: int) -> np.ndarray:
    rows = np.arange(k_h) - k_h // 2
    cols = np.arange(k_w) - k_w // 2
    out = np.empty((k_h * k_w, 2), dtype=np.int64)
    out[:, 0] = np.repeat(rows, k_w)
    out[:, 1] = np.tile(cols, k_h)
    return out


# kernels.py:63-68
def taps(weights: np.ndarray) -> np.ndarray:
    co, ci, kh, kw = weights.shape
    return np.ascontiguousarray(
        np.asarray(weights, dtype=np.float64).reshape(co, ci, kh * kw).transpose(2, 0, 1))


# kernels.py:126-134
def grid_frequencies(n: int, m: int) -> np.ndarray:
    i = np.repeat(np.arange(n), m)
    j = np.tile(np.arange(m), n)
    freqs = np.empty((n * m, 2))
    freqs[:, 0] = i / n
    freqs[:, 1] = j / m
    return freqs


def symbol_field(weights, n=None, m=None, freqs=None, nthreads=0) -> np.ndarray:
    """(F, c_out, c_in) complex128 symbol blocks (symbol.py:108-137)."""
    w = np.asarray(weights, dtype=np.float64)
    co, ci, kh, kw = w.shape
    if freqs is None:
        freqs = grid_frequencies(n, m)
    freqs = np.ascontiguousarray(freqs, dtype=np.float64)
    offs = np.ascontiguousarray(offsets(kh, kw).astype(np.float64))
    tp = taps(w)
    out = np.zeros((len(freqs), co, ci), dtype=np.complex128)
    lib().orc_symbol_blocks(_ptr(freqs), len(freqs), _ptr(offs), kh * kw, _ptr(tp),
                            co, ci, _ptr(out.view(np.float64)), int(nthreads))
    return out


def _work(blocks):
    blocks = np.asarray(blocks)
    F, co, ci = blocks.shape
    wide = co < ci
    work = blocks.conj().transpose(0, 2, 1) if wide else blocks
    return np.ascontiguousarray(work), wide


def svd_values(blocks, tol=DEFAULT_TOL, max_sweeps=DEFAULT_MAX_SWEEPS, nthreads=0,
               return_sweeps=False, f32=False):
    """Per-block singular values, descending, shape (F, min(co,ci)).

    blocksvd.py:253-264.  ``f32=True`` runs the complex64-storage variant
    (study only, not a parity reference)."""
    work, _ = _work(blocks)
    F, mr, nc = work.shape
    sig = np.empty((F, nc))
    fail = np.zeros(F, dtype=np.int8)
    sweeps = np.zeros(F, dtype=np.int32)
    if f32:
        w = np.ascontiguousarray(work.astype(np.complex64))
        fn = lib().orc_svd_values_batch_f32acc if f32 == "acc" else lib().orc_svd_values_batch_f32
        fn(_ptr(w.view(np.float32), _fp), F, mr, nc, tol, max_sweeps, _ptr(sig), _ptr(fail, _i8p),
                                       _ptr(sweeps, _i32p), int(nthreads))
    else:
        w = np.ascontiguousarray(work.astype(np.complex128))
        lib().orc_svd_values_batch(_ptr(w.view(np.float64)), F, mr, nc, tol, max_sweeps,
                                   _ptr(sig), _ptr(fail, _i8p), _ptr(sweeps, _i32p),
                                   int(nthreads))
    out = np.ascontiguousarray(sig[:, ::-1])
    if return_sweeps:
        return out, fail, sweeps
    return out, fail


def _complete_zero_columns(U, sigma):
    # blocksvd.py:184-198
    bad = np.nonzero(~(sigma > 0).all(axis=1))[0]
    for f in bad:
        mat = U[f]
        mr = mat.shape[0]
        for j in np.nonzero(~(sigma[f] > 0))[0]:
            for t in range(mr):
                cand = np.zeros(mr, dtype=np.complex128)
                cand[t] = 1.0
                cand -= mat @ (mat.conj().T @ cand)
                norm = np.linalg.norm(cand)
                if norm > 0.5:
                    mat[:, j] = cand / norm
                    break


def svd_full(blocks, tol=DEFAULT_TOL, max_sweeps=DEFAULT_MAX_SWEEPS, nthreads=0):
    """(U (F,co,r), sigma (F,r) descending, V (F,ci,r), fail (F,)).

    blocksvd.py:201-210 (_finish_full) and :266-270 (wide swap)."""
    work, wide = _work(blocks)
    F, mr, nc = work.shape
    w = np.ascontiguousarray(work.astype(np.complex128))
    Bout = np.empty((F, mr, nc), dtype=np.complex128)
    Vout = np.empty((F, nc, nc), dtype=np.complex128)
    sig = np.empty((F, nc))
    fail = np.zeros(F, dtype=np.int8)
    sweeps = np.zeros(F, dtype=np.int32)
    lib().orc_svd_full_batch(_ptr(w.view(np.float64)), F, mr, nc, tol, max_sweeps,
                             _ptr(Bout.view(np.float64)), _ptr(Vout.view(np.float64)),
                             _ptr(sig), _ptr(fail, _i8p), _ptr(sweeps, _i32p),
                             int(nthreads))
    order = np.argsort(-sig, axis=1, kind="stable")
    sig = np.take_along_axis(sig, order, axis=1)
    Bout = np.take_along_axis(Bout, order[:, None, :], axis=2)
    Vout = np.take_along_axis(Vout, order[:, None, :], axis=2)
    denom = np.where(sig > 0, sig, 1.0)
    U = Bout / denom[:, None, :]
    _complete_zero_columns(U, sig)
    if wide:
        U, Vout = Vout, U
    return U, sig, Vout, fail


def sort_descending(values):
    # blocksvd.py:69-72
    order = np.argsort(-values, kind="stable")
    return values[order]


def spectrum_values(weights, n, m, tol=DEFAULT_TOL, max_sweeps=DEFAULT_MAX_SWEEPS,
                    nthreads=0):
    """compute_spectrum(kernel, dims).values restated (pipeline.py:61-69)."""
    fld = symbol_field(weights, n, m, nthreads=nthreads)
    sig, fail = svd_values(fld, tol, max_sweeps, nthreads)
    if fail.any():
        raise RuntimeError(f"oracle: no convergence at frequency {int(np.argmax(fail))}")
    return sort_descending(np.ascontiguousarray(sig).ravel())


def summary(values):
    """analysis.py:35-53: (max, min, count, condition, mean, hist, edges)."""
    v = np.asarray(values, dtype=np.float64).ravel()
    if v.size == 0:
        raise ValueError("empty spectrum")
    hi, lo = float(v.max()), float(v.min())
    top = hi if hi > 0 else 1.0
    hist, edges = np.histogram(v, bins=64, range=(0.0, top))
    cond = hi / lo if lo > 0 else np.inf
    return hi, lo, v.size, cond, float(v.mean()), hist, edges


def w1(a, b):
    """analysis.py:56-74: both descending; the shorter resampled at the
    longer one's quantile positions t = j/(L-1) by linear interpolation."""
    x = np.sort(np.asarray(a, dtype=np.float64).ravel())[::-1]
    y = np.sort(np.asarray(b, dtype=np.float64).ravel())[::-1]
    if x.size == 0 or y.size == 0:
        raise ValueError("empty spectrum")
    if x.size < y.size:
        x, y = y, x
    if y.size < x.size:
        pos_long = np.linspace(0.0, 1.0, x.size)
        pos_short = np.linspace(0.0, 1.0, y.size)
        y = np.interp(pos_long, pos_short, y[::-1])[::-1]
    return float(np.abs(x - y).mean())
