"""Run one config layer's K1 + batched SVD over a representative sub-range.

python tools/prof_case.py CFG [COUNT] [--layer L] [--values] [--f64] [--reps N]
Prints device time per stage (CUDA events) and per-matrix / per-round costs.
Used for ncu captures (small COUNT keeps the profiled kernel short).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2506_05617_b200 import configs, engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("count", type=int, nargs="?", default=0)
ap.add_argument("--layer", type=int, default=0)
ap.add_argument("--values", action="store_true", help="values only even if the config wants vectors")
ap.add_argument("--f64", action="store_true")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()

wl = configs.WORKLOADS[a.cfg]
layer = wl.layers[a.layer]
dt = "f64" if a.f64 else "f32"
dev = torch.device("cuda:0")
w = configs.layer_weights(layer)
wd = torch.from_numpy(w.astype("float64") if a.f64 else w).to(dev)
F_u = engine.half_grid_count(layer.n, layer.m)
count = a.count or F_u
vec = wl.vectors and not a.values
blocks = engine.symbol_field(wd, layer.n, layer.m, dt, half=True, f_first=0, f_count=count)
for rep in range(a.reps):
    tm = engine.Timer(dev)
    tm.mark("a")
    out = engine.batched_svd(blocks, dt, vec, complete=False)
    tm.mark("b")
    t = tm.seconds("a", "b")
    info = out.info.cpu().numpy()
    rounds = (info.astype("float64") * (min(layer.c_out, layer.c_in) - 1)).sum()
    print(f"cfg{a.cfg} l{a.layer} {dt} vec={vec} count={count}: svd {t * 1e3:.3f} ms, "
          f"sweeps mean {info.mean():.2f}, {t / count * 1e6:.2f} us/matrix, "
          f"{t / rounds * 1e9:.1f} ns per matrix-round (device-wide)", flush=True)
