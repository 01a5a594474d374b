"""Warm start study on the GPU: cold vs warm chains of depth 1..3.

python tools/warmtest.py CFG [CFG ...]
Prints SVD time, sweep statistics, parity vs the golden sigma and factor quality.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "tests/golden/golden.npz"))
dev = torch.device("cuda:0")
for c in [int(x) for x in sys.argv[1:]]:
    wl = configs.WORKLOADS[c]
    layer = wl.layers[0]
    wd = torch.from_numpy(configs.layer_weights(layer)).to(dev)
    blocks = engine.symbol_field(wd, layer.n, layer.m, "f32", half=True)
    for warm, depth in ((False, 0), (True, 1), (True, 2), (True, 3)):
        engine.WARM_DEPTH = max(depth, 1)
        tm = engine.Timer(dev)
        res = lfa_device(wd, layer.n, layer.m, "f32", wl.vectors, timer=tm, warm_start=warm)
        torch.cuda.synchronize()
        t = tm.seconds("t1", "t2")
        info = res.info.cpu().numpy()
        key = f"cfg{c}_l0"
        rep_of, _ = engine.partner_map(layer.n, layer.m)
        sig = res.sigma.cpu().numpy()[rep_of[g[key + "_fidx"]]]
        ref = g[key + "_sigma"]
        err = (np.abs(sig - ref).max(axis=1) / ref[:, 0]).max()
        q = 0.0
        if res.U is not None:
            F_u = blocks.shape[0]
            for u in np.unique(np.linspace(0, F_u - 1, 16).astype(int)):
                U = res.U[u].cpu().numpy().astype(np.complex128)
                V = res.V[u].cpu().numpy().astype(np.complex128)
                s = res.sigma[u].cpu().numpy()
                A = blocks[u].cpu().numpy()
                q = max(q, np.abs((U * s) @ V.conj().T - A).max() / s[0],
                        np.abs(V.conj().T @ V - np.eye(V.shape[1])).max())
        print(f"cfg{c} warm={warm} depth={depth}: svd {t * 1e3:.1f} ms sweeps mean "
              f"{info.mean():.2f} [{info.min()},{info.max()}] parity {err:.2e} "
              f"factors {q:.2e}", flush=True)
