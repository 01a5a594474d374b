"""cfg4 (16 ResNet-18 layers, sigma only) per-shape split: times each block
shape's four layers alone (one lfa_device_multi call per shape) and all 16
together.  python tools/cfg4_prof.py [REPS]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2506_05617_b200 as cs  # noqa: E402
from paper_2506_05617_b200 import configs, engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda:0")
wl = configs.WORKLOADS[4]
items = [(torch.from_numpy(configs.layer_weights(l)).to(dev), l.n, l.m, l) for l in wl.layers]
groups = {}
for w, n, m, l in items:
    groups.setdefault((l.c_out, l.c_in, n, m), []).append((w, n, m))
groups["all"] = [(w, n, m) for w, n, m, _ in items]
for key, g in groups.items():
    best = 1e9
    for _ in range(reps):
        tm = engine.Timer(dev)
        res = cs.lfa_device_multi(g, "f32", False, timer=tm)
        torch.cuda.synchronize()
        best = min(best, tm.seconds("t1", "t2"))
    info = torch.cat([r.info for r in res]).float()
    print(f"{key}: svd {best * 1e3:.1f} ms, sweeps {info.mean().item():.2f}, blocks {info.numel()}", flush=True)
