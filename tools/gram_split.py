"""Per-phase cycle split of the Gram-blocked vs scalar cross phase (cfg5 shape).

Needs an experiment build:  CS_AB_FLAGS=-DCS_PHASE_CLOCKS tools/ab_build.sh clk
    CS_LIBPATH=ab_libs/libclk.so python tools/gram_split.py [COUNT]
Runs the cfg5 batch cold with CS_GRAM=1 and with the default scalar path and
prints the summed CTA cycles per phase (thread 0 of every CTA)."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import _lib, configs, engine  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 240
lib = _lib.load()
fn = lib.cs_debug_phase_cycles
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
buf = (ctypes.c_ulonglong * 8)()
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
w = torch.from_numpy(configs.layer_weights(layer)).to(dev)
blocks = engine.symbol_field(w, layer.n, layer.m, "f32", half=True, f_first=0, f_count=count)
for mode in ("1", "0"):
    os.environ["CS_GRAM"] = mode
    fn(buf, 1)
    tm = engine.Timer(dev)
    tm.mark("a")
    out = engine.batched_svd(blocks, "f32", True)
    tm.mark("b")
    fn(buf, 1)
    c = list(buf)
    tot = sum(c[:5])
    print(f"CS_GRAM={mode}: {tm.seconds('a', 'b') * 1e3:.1f} ms, sweeps {out.info.float().mean().item():.2f}; "
          f"cycles gram {c[0]:.3e} inner {c[1]:.3e} update {c[2]:.3e} within {c[3]:.3e} "
          f"scalar-cross {c[4]:.3e}", flush=True)
