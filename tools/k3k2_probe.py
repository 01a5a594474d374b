"""K3 (tensor-core kernel) and K2 (CS_TCB=0) against the fp64 solve on a warm-started cfg5 sub-range:
python tools/k3k2_probe.py [COUNT ...]"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine
from paper_2506_05617_b200.pipeline import lfa_device
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
for count in [int(a) for a in sys.argv[1:]] or [432, 1024]:
    os.environ.pop("CS_TCB", None)
    k3 = lfa_device(w, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=True, assemble=False)
    os.environ["CS_TCB"] = "0"
    k2 = lfa_device(w, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=True, assemble=False)
    os.environ.pop("CS_TCB", None)
    r = lfa_device(w.double(), layer.n, layer.m, "f64", False, u0=0, count=count, warm_start=False, assemble=False)
    s3, s2, sr = k3.sigma.cpu().numpy(), k2.sigma.cpu().numpy(), r.sigma.cpu().numpy()
    for name, s in (("K3", s3), ("K2", s2)):
        e = np.abs(s - sr).max(axis=1) / sr[:, 0]
        print(count, name, "vs f64: max", e.max(), "argmax", int(e.argmax()), "p50", np.median(e), "p99", np.quantile(e, 0.99),
              "bad(>1e-6)", int((e > 1e-6).sum()), "sweeps", s is s3 and k3.info.float().mean().item() or k2.info.float().mean().item(), flush=True)
    e = np.abs(s2 - sr).max(axis=1) / sr[:, 0]
    print("  K2 bad idx", np.nonzero(e > 1e-6)[0][:20])
    e = np.abs(s3 - sr).max(axis=1) / sr[:, 0]
    print("  K3 bad idx", np.nonzero(e > 1e-6)[0][:20])
