"""Orthonormality of the right factors as a function of warm-start chain depth
(cfg5, fp32 via K3 and fp64 via the warm-started panel kernel):
max |V^H V - I| and max |U^H U - I| over 16 representatives per BFS stage of
the whole-grid warm plan.   python tools/orth_by_depth.py [f32|f64] > profiles/...txt"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402

dt = sys.argv[1] if len(sys.argv) > 1 else "f32"
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
w = w if dt == "f32" else w.double()
res = lfa_device(w, layer.n, layer.m, dt, True)
F = engine.half_grid_count(layer.n, layer.m)
stage = np.zeros(F, dtype=np.int64)
for d, (sel, pred, gsize) in enumerate(engine.subset_plan(layer.n, layer.m, np.arange(F), torch.device("cpu"), None)):
    stage[sel.numpy()] = d
rng = np.random.default_rng(0)
print(f"cfg5 {dt}: orthonormality by warm-chain stage (0 = cold seeds), 16 blocks per stage")
print(f"{'stage':>5} {'blocks':>7} {'max|VhV-I|':>12} {'max|UhU-I|':>12} {'mean sweeps':>12}")
info = res.info.cpu().numpy()
for d in range(stage.max() + 1):
    ids = np.nonzero(stage == d)[0]
    pick = rng.choice(ids, size=min(16, len(ids)), replace=False)
    t = torch.from_numpy(pick).to(dev)
    V = res.V[t].cpu().numpy().astype(np.complex128)
    U = res.U[t].cpu().numpy().astype(np.complex128)
    ov = max(np.abs(v.conj().T @ v - np.eye(v.shape[1])).max() for v in V)
    ou = max(np.abs(u.conj().T @ u - np.eye(u.shape[1])).max() for u in U)
    print(f"{d:>5} {len(ids):>7} {ov:>12.3e} {ou:>12.3e} {info[ids].mean():>12.2f}", flush=True)
