import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN_PATH)


@pytest.fixture(scope="session")
def orc():
    from oracle import oracle

    return oracle


@pytest.fixture(scope="session")
def cuda():
    """The gpu tests never skip: on the GPU box a missing device is a failure."""
    import torch

    assert torch.cuda.is_available(), "gpu-marked test run without a CUDA device"
    from paper_2506_05617_b200 import _lib

    _lib.load()
    return torch.device("cuda", 0)


def averaging_symbol(k1, k2):
    # pkg/tests/conftest.py:19-21 closed form
    return (1.0 + 2.0 * np.cos(2 * np.pi * k1)) * (1.0 + 2.0 * np.cos(2 * np.pi * k2)) / 9.0


def identity_kernel(channels):
    import paper_2506_05617_b200 as cs

    w = np.zeros((channels, channels, 1, 1))
    w[:, :, 0, 0] = np.eye(channels)
    return cs.ConvKernel.from_array(w)


def per_freq_rel_err(sig, ref):
    """max_j |sigma - sigma_ref| / sigma_ref[f, 0], per frequency (SURVEY 8(c) bar)."""
    sig = np.asarray(sig)
    ref = np.asarray(ref)
    scale = np.maximum(ref[:, :1], 1e-300)
    return np.abs(sig - ref).max(axis=1) / scale[:, 0]
