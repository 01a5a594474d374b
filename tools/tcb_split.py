"""Per-phase cycle split of the tensor-core blocked kernel (CS_TCB_CLOCKS build):
CS_LIBPATH=ab_libs/libtcbclk.so python tools/tcb_split.py [COUNT] [WARM]"""
import ctypes, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import _lib, configs  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402
count = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
warm = (sys.argv[2] != "0") if len(sys.argv) > 2 else False
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
wd = torch.from_numpy(configs.layer_weights(layer)).to(dev)
L = _lib.load()
buf = (ctypes.c_ulonglong * 32)()
lfa_device(wd, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=warm, assemble=False)
L.cs_debug_tcb_cycles(buf, 1)
sb = (ctypes.c_ulonglong * 64)()
has_sw = hasattr(L, 'cs_debug_tcb_sweeps')
if has_sw:
    L.cs_debug_tcb_sweeps(sb, 1)
res = lfa_device(wd, layer.n, layer.m, "f32", True, u0=0, count=count, warm_start=warm, assemble=False)
L.cs_debug_tcb_cycles(buf, 0)
n = buf[9]
names = ["gram", "G-read", "angles", "D (rot/exp)", "bop+update", "epi-add+V-wait", "exchange", "wait incoming X"]
tot = sum(buf[i] for i in range(8))
print(f"{count} blocks warm={warm}: {n} super-rounds on CTA thread 0s, sweeps {res.info.float().mean().item():.2f}")
for i, nm in enumerate(names):
    print(f"  {nm:12s} {buf[i] / n:8.0f} cycles/super-round ({100 * buf[i] / tot:.1f}%)")
print(f"  total        {tot / n:8.0f}")
nm = max(buf[13], 1)
print(f"  per matrix: load {buf[10] / nm:.0f}, verdicts {buf[11] / nm:.0f}, epilogue {buf[12] / nm:.0f} cycles "
      f"({n / nm:.1f} super-rounds per matrix -> {(buf[10] + buf[11] + buf[12]) / n:.0f} per super-round)")
print(f"  rotating super-rounds: {buf[14] / n:.3f} product form, {buf[15] / n:.3f} exp form")
print(f"  exp form: {buf[16] / max(buf[15], 1):.0f} cycles per call")
print(f"  product form: {buf[17] / max(buf[14], 1):.0f} cycles per cross call (all product-form calls: {buf[14]}), full {buf[18]}")
ru = max(buf[14] + buf[15], 1)
print(f"  update per rotating super-round: bop+finish_v {buf[19] / ru:.0f}, MMA waits {buf[20] / ru:.0f}, "
      f"lo staging {buf[21] / ru:.0f}, issue+epi {buf[22] / ru:.0f}")
nx = max(n - nm * 7, 1)  # exchanges (the last super-round of a sweep has none; ~7 sweeps per matrix)
print(f"  exchange split per exchange: outbox copy + CTA barrier {buf[23] / nx:.0f}, fence + publish {buf[24] / nx:.0f}, "
      f"wait for the sender {buf[25] / nx:.0f} (not ready on arrival: {buf[28] / nx:.3f}), meta read {buf[26] / nx:.0f}")
print(f"  sparse rotating super-rounds (rotations applied in place): {buf[29] / n:.3f} of all, {buf[30] / max(buf[29], 1):.0f} cycles each")
if has_sw:
    L.cs_debug_tcb_sweeps(sb, 0)
    print("  by sweep: cycles per super-round, share of all cycles, dense / sparse rotating fraction, super-rounds per matrix")
    allc = max(sum(sb[i] for i in range(16)), 1)
    for i in range(16):
        if sb[16 + i]:
            print(f"    sweep {i + 1:2d}: {sb[i] / sb[16 + i]:7.0f}  {100 * sb[i] / allc:5.1f}%  dense {sb[32 + i] / sb[16 + i]:.3f} "
                  f"sparse {sb[48 + i] / sb[16 + i]:.3f}  {sb[16 + i] / nm:6.2f}")
