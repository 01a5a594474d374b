"""Small warm-started cfg5 solve for profiling the tensor-core Jacobi kernel:
python tools/tcb_prof.py [COUNT]  (ncu -k regex:jacobi_tcb ...)"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 1200
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
wd = torch.from_numpy(configs.layer_weights(layer)).to(dev)
for _ in range(2):
    tm = engine.Timer(dev)
    res = lfa_device(wd, layer.n, layer.m, "f32", True, u0=0, count=count, timer=tm, warm_start=True,
                     assemble=False)
    torch.cuda.synchronize()
    print(f"{count} blocks: svd {tm.seconds('t1', 't2') * 1e3:.1f} ms, sweeps {res.info.float().mean().item():.2f}",
          flush=True)
