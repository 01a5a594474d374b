"""The C-ABI shared library: builds for sm_100a, loads without a GPU, exports
every entry point include/convspectra_b200.h declares, and rejects bad
arguments with the documented status codes before touching CUDA."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2506_05617_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "convspectra_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIBPATH):
        _build.build()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(cs_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_path():
    syms = declared_symbols()
    for s in ("cs_symbol_field", "cs_batched_svd", "cs_batched_svd_grouped",
              "cs_spectrum_values", "cs_last_error_string"):
        assert s in syms


def test_every_declared_symbol_is_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIBPATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cs_[a-z0-9_]+)\b", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # and the ctypes binding covers exactly the declared surface
    assert sorted(_lib.EXPORTED) == declared_symbols()


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIBPATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_grid_count(lib):
    assert lib.cs_abi_version() == 1
    assert lib.cs_half_grid_count(256, 256) == 32770
    assert lib.cs_half_grid_count(5, 3) == 8
    assert lib.cs_half_grid_count(0, 3) == 0


def test_invalid_arguments_return_einval(lib):
    st = lib.cs_symbol_field(None, 0, 1, 1, 3, 3, 4, 4, 0, 1, 1, None, 0, None)
    assert st == _lib.CS_EINVAL and "null" in _lib.last_error()
    p = ctypes.c_void_p(16)
    st = lib.cs_symbol_field(p, 0, 0, 1, 3, 3, 4, 4, 0, 1, 1, p, 0, None)
    assert st == _lib.CS_EINVAL and "dimensions" in _lib.last_error()
    st = lib.cs_symbol_field(p, 0, 1, 1, 3, 3, 4, 4, 0, 100, 1, p, 0, None)
    assert st == _lib.CS_EINVAL and "range" in _lib.last_error()
    st = lib.cs_batched_svd(p, 7, 1, 2, 2, 0, 1e-13, 100, p, None, None, p, None, None, 0, None)
    assert st == _lib.CS_EINVAL and "dtype" in _lib.last_error()
    st = lib.cs_batched_svd(p, 0, 1, 2, 2, 1, 1e-13, 100, p, None, None, p, None, None, 0, None)
    assert st == _lib.CS_EINVAL
    st = lib.cs_batched_svd(p, 0, 1, 2, 2, 0, 1e-13, 0, p, None, None, p, None, None, 0, None)
    assert st == _lib.CS_EINVAL and "max_sweeps" in _lib.last_error()
    # an empty batch is a no-op
    assert lib.cs_batched_svd(None, 0, 0, 2, 2, 0, 1e-13, 100, None, None, None, None, None,
                              None, 0, None) == _lib.CS_OK


def test_status_mapping():
    import paper_2506_05617_b200 as cs

    with pytest.raises(cs.AllocationFailure):
        _lib.check(_lib.CS_ENOMEM, "x")
    with pytest.raises(cs.ConvergenceFailure):
        _lib.check(_lib.CS_ENOCONV, "x")
    with pytest.raises(RuntimeError):
        _lib.check(_lib.CS_ECUDA, "x")
    _lib.check(_lib.CS_OK)
