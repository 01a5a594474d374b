"""Golden files for the NPY/CSV row, written by the
REFERENCE's own npyio (pkg/src/convspectra/npyio.py), imported read-only
from /root/reference in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden_io.py

Writes tests/golden/io/: kernel_f32.npy, kernel_f64.npy (write_npy_kernel of
seeded random kernels), spectrum.csv (write_spectrum_csv of a fixed value
set incl. ties, zeros and values needing all 17 digits).  Nothing on the GPU
box reads /root/reference.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from convspectra import kernels as rk  # noqa: E402
from convspectra import npyio as rio  # noqa: E402

out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "io")
os.makedirs(out, exist_ok=True)
k64 = rk.random_kernel(3, 2, 3, 5, seed=11)
k32 = rk.ConvKernel(weights=k64.weights.astype(np.float32).astype(np.float64), precision="f32")
rio.write_npy_kernel(os.path.join(out, "kernel_f64.npy"), k64)
rio.write_npy_kernel(os.path.join(out, "kernel_f32.npy"), k32)
vals = np.array([np.pi, 2.0, 2.0, 1.0 / 3.0, 1e-300, 0.0, 123456789.123456789, 5e-324])
rio.write_spectrum_csv(vals, os.path.join(out, "spectrum.csv"))
np.save(os.path.join(out, "weights_f64.npy"), k64.weights)
print("wrote", sorted(os.listdir(out)))
