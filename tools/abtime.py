"""Same-box A/B timing of the LFA SVD phase (cfg5 by default).

python tools/abtime.py [CFG] [REPS]   (select a library with CS_LIBPATH=...)
Prints min SVD-phase time for cold and warm starts.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
wl = configs.WORKLOADS[cfg]
layer = wl.layers[0]
wd = torch.from_numpy(configs.layer_weights(layer)).to(dev)
lib = os.environ.get("CS_LIBPATH", "default")
for warm in (False, True):
    best, sweeps = 1e9, 0.0
    for _ in range(reps):
        tm = engine.Timer(dev)
        res = lfa_device(wd, layer.n, layer.m, "f32", wl.vectors, timer=tm, warm_start=warm)
        torch.cuda.synchronize()
        best = min(best, tm.seconds("t1", "t2"))
        sweeps = res.info.float().mean().item()
    print(f"{os.path.basename(lib)} cfg{cfg} warm={warm}: svd {best * 1e3:.1f} ms sweeps {sweeps:.3f}",
          flush=True)
