"""Matrix-free periodic convolution operator.

``apply_conv(kernel, x, dims)`` applies the unrolled periodic stride-1
convolution without materialising it (the reference's explicit.py:149-178,
apply_conv_reference, periodic boundary), on the device (cs_apply_conv).
With the global singular vectors of ``materialize_singular_vector`` it checks
||A v - sigma u|| at sizes where the dense matrix cannot exist.
"""

from __future__ import annotations

import numpy as np

from . import engine
from .kernels import ConvKernel, SpatialDims, validate_kernel


def apply_conv(kernel: ConvKernel, x, dims: SpatialDims, *, device=None, dtype=None):
    """y = A x for x of shape (m, n, c_in) (or flat, index (x1*n + x2)*c_in + ch).

    Returns a device tensor (m, n, c_out) for device input, numpy otherwise."""
    validate_kernel(kernel)
    dev = engine.require_cuda(device if device is not None else
                              (x.device if hasattr(x, "device") and
                               getattr(x.device, "type", "") == "cuda" else None))
    dt = dtype or kernel.precision
    torch = engine.torch
    is_np = isinstance(x, np.ndarray)
    xt = torch.as_tensor(np.ascontiguousarray(x)) if is_np else x
    xt = xt.to(dev).reshape(dims.m, dims.n, kernel.c_in).to(engine.complex_dtype(dt))
    w = engine.weights_to_device(kernel, dt, dev)
    y = engine.apply_conv(w, xt, dims.n, dims.m, dt)
    return y.cpu().numpy() if is_np else y
