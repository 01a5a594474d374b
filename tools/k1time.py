"""Device time of K1 (half-grid assembly) for a config: python tools/k1time.py [CFG] [REPS]."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[cfg].layers[0]
w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
out = engine.symbol_field(w, layer.n, layer.m, "f32", half=True)
best = 1e9
for _ in range(reps):
    tm = engine.Timer(dev)
    tm.mark("a")
    engine.symbol_field(w, layer.n, layer.m, "f32", half=True, out=out)
    tm.mark("b")
    best = min(best, tm.seconds("a", "b"))
nbytes = out.numel() * 8
print(f"{os.path.basename(os.environ.get('CS_LIBPATH', 'default'))} cfg{cfg} K1 {best * 1e3:.3f} ms "
      f"{nbytes / best / 1e9:.0f} GB/s")
