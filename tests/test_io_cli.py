"""NPY / CSV / CLI row against files written by the
reference's own npyio (tests/golden/make_golden_io.py), the reference's
error taxonomy for malformed files (T/test_npyio.py), and the CLI contract
(CS/cli.py: exit codes 0/2/3/4)."""

import json
import os
import struct

import numpy as np
import pytest

import paper_2506_05617_b200 as cs
from paper_2506_05617_b200 import cli, npyio

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def test_read_reference_npy_files():
    w = np.load(os.path.join(GOLD, "weights_f64.npy"))
    k64 = npyio.read_npy_kernel(os.path.join(GOLD, "kernel_f64.npy"))
    assert k64.precision == "f64" and np.array_equal(k64.weights, w)
    k32 = npyio.read_npy_kernel(os.path.join(GOLD, "kernel_f32.npy"))
    assert k32.precision == "f32" and k32.weights.dtype == np.float64
    assert np.array_equal(k32.weights, w.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("name", ["kernel_f64.npy", "kernel_f32.npy"])
def test_write_npy_bytes_match_reference(tmp_path, name):
    k = npyio.read_npy_kernel(os.path.join(GOLD, name))
    dst = tmp_path / name
    npyio.write_npy_kernel(dst, k)
    assert dst.read_bytes() == open(os.path.join(GOLD, name), "rb").read()
    assert len(dst.read_bytes()) % 64 == (k.weights.size * (4 if k.precision == "f32" else 8)) % 64


def test_npy_readable_by_numpy(tmp_path):
    k = cs.random_kernel(2, 3, 3, 3, seed=4)
    npyio.write_npy_kernel(tmp_path / "k.npy", k)
    assert np.array_equal(np.load(tmp_path / "k.npy"), k.weights)


def _npy(header: str, payload: bytes, version=b"\x01\x00", magic=npyio.MAGIC) -> bytes:
    h = header.encode("latin1")
    return magic + version + struct.pack("<H", len(h)) + h + payload


@pytest.mark.parametrize("blob,exc", [
    (b"NOTNPY" + b"\x00" * 20, cs.BadMagic),
    (_npy("{'descr': '<f8', 'fortran_order': False, 'shape': (1, 1, 1, 1), }\n", b"\x00" * 8,
          version=b"\x02\x00"), cs.BadMagic),
    (_npy("{'descr': '<i4', 'fortran_order': False, 'shape': (1, 1, 1, 1), }\n", b"\x00" * 4),
     cs.UnsupportedDescr),
    (_npy("{'descr': '>f8', 'fortran_order': False, 'shape': (1, 1, 1, 1), }\n", b"\x00" * 8),
     cs.UnsupportedDescr),
    (_npy("{'descr': '<f8', 'fortran_order': True, 'shape': (1, 1, 1, 1), }\n", b"\x00" * 8),
     cs.FortranOrderUnsupported),
    (_npy("{'descr': '<f8', 'fortran_order': False, 'shape': (2, 2), }\n", b"\x00" * 32),
     cs.ShapeRankNot4),
    (_npy("{'descr': '<f8', 'fortran_order': False, 'shape': (2, 2, 1, 1), }\n", b"\x00" * 31),
     cs.TruncatedPayload),
    (npyio.MAGIC + b"\x01\x00" + struct.pack("<H", 200) + b"{", cs.TruncatedPayload),
    (_npy("{'descr': '<f8', 'fortran_order': False, 'shape': (1, 1, 1, 1), \n", b"\x00" * 8), cs.BadMagic),
])
def test_malformed_npy_raises_reference_errors(tmp_path, blob, exc):
    p = tmp_path / "bad.npy"
    p.write_bytes(blob)
    with pytest.raises(exc):
        npyio.read_npy_kernel(p)


def test_nonfinite_weights_rejected(tmp_path):
    w = np.ones((1, 1, 2, 2))
    w[0, 0, 1, 0] = np.nan
    npyio.write_npy_kernel(tmp_path / "n.npy", w)
    with pytest.raises(cs.NonFiniteWeight):
        npyio.read_npy_kernel(tmp_path / "n.npy")


def test_spectrum_csv_matches_reference(tmp_path):
    vals = np.array([np.pi, 2.0, 2.0, 1.0 / 3.0, 1e-300, 0.0, 123456789.123456789, 5e-324])
    npyio.write_spectrum_csv(vals, tmp_path / "s.csv")
    assert (tmp_path / "s.csv").read_text() == open(os.path.join(GOLD, "spectrum.csv")).read()
    back = npyio.read_spectrum_csv(tmp_path / "s.csv")
    assert np.array_equal(back, vals)


def test_cli_gen_kernel_and_usage_errors(tmp_path):
    out = tmp_path / "k.npy"
    assert cli.main(["gen-kernel", "--cout", "4", "--cin", "3", "--seed", "2", "--out", str(out)]) == 0
    k = npyio.read_npy_kernel(out)
    assert np.array_equal(k.weights, cs.random_kernel(4, 3, 3, 3, seed=2).weights)
    assert cli.main(["singvals"]) == 2  # missing required arguments
    assert cli.main(["singvals", "--weights", str(tmp_path / "missing.npy"), "--height", "4",
                     "--width", "4"]) == 2  # OSError -> usage/validation


def test_cli_without_cuda_exits_3(tmp_path, monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    npyio.write_npy_kernel(tmp_path / "k.npy", cs.random_kernel(2, 2, 3, 3, seed=1))
    assert cli.main(["singvals", "--weights", str(tmp_path / "k.npy"), "--height", "4", "--width", "4",
                     "--out", str(tmp_path / "s.csv")]) == 3


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,bar", [("f64", 1e-10), ("f32", 1e-5)])
def test_cli_singvals_on_gpu(tmp_path, orc, dtype, bar):
    k = cs.random_kernel(3, 2, 3, 3, seed=5)
    npyio.write_npy_kernel(tmp_path / "k.npy", k)
    rc = cli.main(["singvals", "--weights", str(tmp_path / "k.npy"), "--height", "6", "--width", "5",
                   "--dtype", dtype, "--out", str(tmp_path / "s.csv"), "--meta", str(tmp_path / "m.json")])
    assert rc == 0
    vals = npyio.read_spectrum_csv(tmp_path / "s.csv")
    ref = orc.spectrum_values(k.weights, 5, 6)
    assert vals.shape == ref.shape
    assert np.abs(vals - ref).max() <= bar * ref[0]
    meta = json.load(open(tmp_path / "m.json"))
    assert meta["sv_count"] == len(ref) and meta["dims"] == {"n": 5, "m": 6} and meta["dtype"] == dtype
