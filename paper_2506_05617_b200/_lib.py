"""ctypes binding of the C-ABI in include/convspectra_b200.h.

The product path has exactly one backend: the sm_100a library built from
csrc/.  There is no CPU fallback -- if the library or a CUDA device is
missing, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import AllocationFailure, ConvergenceFailure, ZeroDimension

_HERE = os.path.dirname(os.path.abspath(__file__))
LIBPATH = os.path.join(_HERE, "lib", "libconvspectra_b200.so")

CS_OK, CS_EINVAL, CS_ENOMEM, CS_ENOCONV, CS_ECUDA = 0, 1, 2, 3, 4
CS_F32, CS_F64 = 0, 1
CS_BLOCK_CONTIGUOUS, CS_FREQUENCY_STRIDED = 0, 1

_lock = threading.Lock()
_LIB = None

_vp = ctypes.c_void_p
_ll = ctypes.c_longlong
_i = ctypes.c_int
_d = ctypes.c_double
_sz = ctypes.c_size_t


class SvdGroup(ctypes.Structure):
    _fields_ = [("blocks", _vp), ("count", _ll), ("c_out", _i), ("c_in", _i),
                ("sigma", _vp), ("U", _vp), ("V", _vp), ("info", _vp), ("zero_sigma", _vp),
                ("tol", _d)]


_SIGNATURES = {
    "cs_abi_version": (_i, []),
    "cs_last_error_string": (ctypes.c_char_p, []),
    "cs_half_grid_count": (_ll, [_i, _i]),
    "cs_symbol_field": (_i, [_vp, _i, _i, _i, _i, _i, _i, _i, _ll, _ll, _i, _vp, _i, _vp]),
    "cs_symbol_at": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _ll, _vp, _vp]),
    "cs_expand_half_grid": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "cs_check_conj_symmetry": (_i, [_vp, _i, _i, _i, _i, _i, _vp, _vp]),
    "cs_batched_svd_workspace": (_sz, [_i, _ll, _i, _i, _i]),
    "cs_batched_svd": (_i, [_vp, _i, _ll, _i, _i, _i, _d, _i, _vp, _vp, _vp, _vp, _vp, _vp,
                            _sz, _vp]),
    "cs_batched_svd_plan_kind": (_i, [_i, _ll, _i, _i, _i]),
    "cs_batched_svd_indexed": (_i, [_vp, _i, _ll, _i, _i, _i, _d, _i, _vp, _vp, _vp, _vp, _ll,
                                    _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "cs_warm_start_gemm": (_i, [_vp, _i, _i, _i, _ll, _vp, _vp, _vp, _vp, _vp]),
    "cs_batched_svd_grouped_workspace": (_sz, [ctypes.POINTER(SvdGroup), _i, _i, _i]),
    "cs_batched_svd_grouped": (_i, [ctypes.POINTER(SvdGroup), _i, _i, _i, _d, _i, _vp, _sz,
                                    _vp]),
    "cs_complete_zero_columns": (_i, [_vp, _i, _ll, _i, _i, _vp, _vp, _vp]),
    "cs_first_failure": (_i, [_vp, _ll, _vp, _vp]),
    "cs_fft_field_workspace": (_sz, [_i, _i, _i, _i, _i]),
    "cs_fft_transform": (_i, [_vp, _i, _i, _i, _i, _i, _i, _i, _vp, _sz, _vp]),
    "cs_fft_gather": (_i, [_vp, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "cs_analysis_workspace": (_sz, [_ll]),
    "cs_spectral_summary": (_i, [_vp, _ll, _vp, _vp, _vp, _vp, _sz, _vp]),
    "cs_sort_descending_f64": (_i, [_vp, _vp, _ll, _vp, _sz, _vp]),
    "cs_wasserstein1_sum": (_i, [_vp, _ll, _vp, _ll, _vp, _vp, _sz, _vp]),
    "cs_spectrum_values_workspace": (_sz, [_ll, _i]),
    "cs_spectrum_values": (_i, [_vp, _i, _ll, _i, _i, _i, _i, _vp, _vp, _sz, _vp]),
    "cs_materialize_vector": (_i, [_vp, _i, _i, _i, _i, _i, _i, _i, _i, _vp, _vp]),
    "cs_apply_conv": (_i, [_vp, _i, _i, _i, _i, _i, _i, _i, _vp, _vp, _vp]),
    "cs_measure_fma_peak": (_d, [_i, _i]),
}

EXPORTED = tuple(_SIGNATURES)


def load(path: str | None = None):
    """Load (once) and return the C-ABI library.  Raises if it is not built."""
    global _LIB
    with _lock:
        if _LIB is not None and path is None:
            return _LIB
        p = path or os.environ.get("CS_LIBPATH") or LIBPATH  # override: A/B builds
        if not os.path.exists(p):
            raise RuntimeError(
                f"convspectra_b200: CUDA library not built ({p}); run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (needs nvcc)")
        lib = ctypes.CDLL(p)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.cs_abi_version() != 1:
            raise RuntimeError("convspectra_b200: ABI version mismatch")
        if path is None:
            _LIB = lib
        return lib


def last_error() -> str:
    msg = load().cs_last_error_string()
    return msg.decode() if msg else ""


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference's exception taxonomy."""
    if status == CS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == CS_EINVAL:
        raise ZeroDimension(msg) if "dimension" in msg else ValueError(msg)
    if status == CS_ENOMEM:
        raise AllocationFailure(msg)
    if status == CS_ENOCONV:
        raise ConvergenceFailure(msg)
    raise RuntimeError(f"CUDA error in {msg}")
