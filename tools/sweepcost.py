"""Cost of one rotation-free (check) sweep vs an average rotating sweep, cfg5 shape.

Orthogonal-column input (A = Q diag(s)) converges in the first sweep, so its
time is load + one check sweep + epilogue.  A slightly perturbed one takes one
small-rotation sweep, then the Gram check (or, with CS_GRAM_CHECK=0, a
rotation-free sweep): the difference of the two settings prices the check."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import engine  # noqa: E402

dev = torch.device("cuda:0")
N, n = 32770 // 4, 256
g = torch.Generator(device="cpu").manual_seed(1)
base = torch.randn(64, n, n, dtype=torch.complex64, generator=g)
q, _ = torch.linalg.qr(base)
s = torch.linspace(3.0, 0.01, n)
orth = (q * s).to(dev)
orth = orth.repeat(N // 64 + 1, 1, 1)[:N].contiguous()
rnd = base.to(dev).repeat(N // 64 + 1, 1, 1)[:N].contiguous()
pert = (orth + 1e-4 * 3.0 * torch.randn_like(orth)).contiguous()
cases = [("orthogonal", orth), ("random", rnd)] if len(sys.argv) < 2 else []
cases.append(("perturbed", pert))
for name, blocks in cases:
    for vec in (False, True):
        best = 1e9
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            out = engine.batched_svd(blocks, "f32", vec)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        sw = out.info.float().mean().item()
        print(f"{name} vectors={vec}: {best:.1f} ms, sweeps {sw:.2f}, per sweep {best / sw:.1f} ms",
              flush=True)
