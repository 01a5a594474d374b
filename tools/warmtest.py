import os, sys, time, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.pipeline import lfa_device
g = np.load("tests/golden/golden.npz")
dev = torch.device("cuda:0")
for c in [int(x) for x in sys.argv[1:]]:
    wl = configs.WORKLOADS[c]; layer = wl.layers[0]
    wd = torch.from_numpy(configs.layer_weights(layer)).to(dev)
    for warm in (False, True):
        for rep in range(2):
            tm = engine.Timer(dev)
            res = lfa_device(wd, layer.n, layer.m, "f32", wl.vectors, timer=tm, warm_start=warm)
            torch.cuda.synchronize()
        t = tm.seconds("t1", "t2")
        info = res.info.cpu().numpy()
        key = f"cfg{c}_l0"
        rep_of, _ = engine.partner_map(layer.n, layer.m)
        fidx = g[key + "_fidx"]
        sig = res.sigma.cpu().numpy()[rep_of[fidx]]
        ref = g[key + "_sigma"]
        err = (np.abs(sig - ref).max(axis=1) / ref[:, 0]).max()
        # vector sanity on a few reps: reconstruction
        rerr = 0.0
        if wl.vectors:
            blocks = engine.symbol_field(wd, layer.n, layer.m, "f32", half=True)
            for u in [0, 1, 2, 100, 101, 102, len(info) - 1]:
                U = res.U[u].cpu().numpy().astype(np.complex128); V = res.V[u].cpu().numpy().astype(np.complex128); s = res.sigma[u].cpu().numpy()
                A = blocks[u].cpu().numpy()
                rerr = max(rerr, np.abs((U * s) @ V.conj().T - A).max() / s[0], np.abs(V.conj().T @ V - np.eye(V.shape[1])).max())
        print(f"cfg{c} warm={warm}: svd {t*1e3:.1f} ms sweeps mean {info.mean():.2f} min {info.min()} max {info.max()} parity {err:.2e} recon/orth {rerr:.2e}", flush=True)
