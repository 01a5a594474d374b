"""Bitwise comparison of two builds of the library on a warm-started cfg5
sub-range (sigma, U, V, sweeps):  python tools/bitwise_ab.py LIB_A LIB_B [COUNT]
(each build runs in its own process; "default" = the in-tree library)."""
import os
import subprocess
import sys

import numpy as np

if len(sys.argv) > 1 and sys.argv[1] == "--run":
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2506_05617_b200 import configs  # noqa: E402
    from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402
    count, out = int(sys.argv[2]), sys.argv[3]
    dev = torch.device("cuda:0")
    layer = configs.WORKLOADS[5].layers[0]
    w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
    r = lfa_device(w, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=True, assemble=False)
    np.savez(out, sigma=r.sigma.cpu().numpy(), U=r.U.cpu().numpy(), V=r.V.cpu().numpy(), info=r.info.cpu().numpy())
    sys.exit(0)

libs = sys.argv[1:3]
count = sys.argv[3] if len(sys.argv) > 3 else "2048"
res = []
for i, lib in enumerate(libs):
    env = dict(os.environ)
    if lib != "default":
        env["CS_LIBPATH"] = lib
    f = f"/tmp/bitwise_ab_{i}.npz"
    subprocess.run([sys.executable, __file__, "--run", count, f], env=env, check=True)
    res.append(np.load(f))
for k in ("sigma", "U", "V", "info"):
    a, b = res[0][k], res[1][k]
    print(k, "bitwise equal" if np.array_equal(a, b) else f"DIFFER max {np.abs(a - b).max():.3e}")
