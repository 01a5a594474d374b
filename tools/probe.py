"""Ad-hoc GPU probe: parity of sampled sigma vs golden + device timing per config."""
import os, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2506_05617_b200 as cs
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.pipeline import lfa_device

g = np.load(os.path.join(ROOT, "tests/golden/golden.npz"))
dev = torch.device("cuda:0")
which = [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]
print("fp32 FFMA peak TF/s", engine.fma_peak_flops("f32") / 1e12, "fp64", engine.fma_peak_flops("f64") / 1e12, flush=True)
for c in which:
    wl = configs.WORKLOADS[c]
    tot_sv = 0
    t_all = 0.0
    for li, layer in enumerate(wl.layers):
        key = f"cfg{c}_l{li}"
        w = configs.layer_weights(layer)
        wd = torch.from_numpy(w).to(dev)
        n, m = layer.n, layer.m
        tm = engine.Timer(dev)
        torch.cuda.synchronize()
        t0 = time.time()
        res = lfa_device(wd, n, m, "f32", wl.vectors, timer=tm)
        torch.cuda.synchronize()
        wall = time.time() - t0
        t_k1 = tm.seconds("t0", "t1"); t_svd = tm.seconds("t1", "t3")
        info = res.info.cpu().numpy()
        tot_sv += layer.sv_count
        t_all += t_k1 + t_svd
        msg = f"{key}: k1 {t_k1*1e3:.3f} ms svd {t_svd*1e3:.3f} ms wall {wall:.3f}s sweeps [{info.min()},{info.max()}] mean {info.mean():.2f}"
        if key + "_sigma" in g.files:
            fidx = g[key + "_fidx"]
            rep_of, _ = engine.partner_map(n, m)
            sig = res.sigma.cpu().numpy()[rep_of[fidx]]
            ref = g[key + "_sigma"]
            err = (np.abs(sig - ref).max(axis=1) / ref[:, 0]).max()
            msg += f" parity max rel {err:.2e}"
        print(msg, flush=True)
    print(f"cfg{c}: {tot_sv} SVs, device time {t_all*1e3:.3f} ms -> {tot_sv/t_all:.3e} SV/s", flush=True)
