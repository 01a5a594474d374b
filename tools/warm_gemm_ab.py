"""Warm-start GEMM (cs_warm_start_gemm) accuracy and time on cfg5-shaped
batches: X_i = A_{wid[i]} V_{sid[i]} against an fp64 product on a sample,
and the device time of one cfg5-sized call (32k items) with CUDA events.
python tools/warm_gemm_ab.py [COUNT]   (library: CS_LIBPATH=...)"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import engine  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
dev = torch.device("cuda:0")
for co, ci in ((256, 256), (256, 128)):
    nb, nv = 64, 48
    rng = np.random.default_rng(co + ci)
    A = (rng.standard_normal((nb, co, ci)) + 1j * rng.standard_normal((nb, co, ci))) / np.sqrt(ci)
    V = (rng.standard_normal((nv, ci, ci)) + 1j * rng.standard_normal((nv, ci, ci))) / np.sqrt(ci)
    A = A.astype(np.complex64); V = V.astype(np.complex64)
    n = 40
    wid = np.array([(7 * i + 3) % nb for i in range(n)], dtype=np.int64)
    sid = np.array([(5 * i + 1) % nv for i in range(n)], dtype=np.int64)
    ref = np.einsum("irk,ikc->irc", A[wid].astype(np.complex128), V[sid].astype(np.complex128))
    bt, vt = torch.from_numpy(A).to(dev), torch.from_numpy(V).to(dev)
    out = torch.empty((n, co, ci), dtype=torch.complex64, device=dev)
    engine.warm_start_gemm(bt, "f32", torch.from_numpy(wid).to(dev), torch.from_numpy(sid).to(dev), vt, out)
    got = out.cpu().numpy().astype(np.complex128)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    bias = float(np.mean((np.abs(got) ** 2).sum(axis=(1, 2)) / (np.abs(ref) ** 2).sum(axis=(1, 2)) - 1))
    print(f"{co}x{ci}: max rel err {err:.3e}, energy bias {bias:.3e}", flush=True)
# timing at cfg5 size: count items over a 32770-block field, seeds among 2048 V's
co = ci = 256
nb, nv = 32770, 2048
blocks = torch.randn((nb, co, ci), dtype=torch.complex64, device=dev) / 16
Vw = torch.randn((nv, ci, ci), dtype=torch.complex64, device=dev) / 16
g = torch.Generator(device="cpu").manual_seed(0)
wid = torch.randperm(nb, generator=g)[:count].to(dev)
sid = torch.randint(0, nv, (count,), generator=g).to(dev)
out = torch.empty((count, co, ci), dtype=torch.complex64, device=dev)
for _ in range(2):
    engine.warm_start_gemm(blocks, "f32", wid, sid, Vw, out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(); engine.warm_start_gemm(blocks, "f32", wid, sid, Vw, out); e1.record()
    torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
fl = 8.0 * count * co * ci * ci
print(f"{count} items 256x256x256: {best:.2f} ms, {fl / best / 1e9:.1f} TFLOP/s (fp32-accurate complex), "
      f"{os.path.basename(os.environ.get('CS_LIBPATH', 'default'))}", flush=True)
