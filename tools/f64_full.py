"""Full cfg5 solve in fp64 (the 1e-10 parity precision): device time, sweeps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402

dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
w = torch.from_numpy(configs.layer_weights(layer).astype("float64")).to(dev)
tm = engine.Timer(dev)
res = lfa_device(w, layer.n, layer.m, "f64", True, timer=tm)
torch.cuda.synchronize()
sv = res.values.numel()
t = tm.seconds("t0", "t3")
print(f"cfg5 fp64 sigma+U+V: {t:.2f} s ({tm.seconds('t1', 't2'):.2f} s SVD), {sv / t / 1e6:.3f}M SV/s, "
      f"sweeps {res.info.float().mean().item():.2f}, converged {(res.info > 0).all().item()}")
