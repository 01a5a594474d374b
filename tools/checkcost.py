"""Price of one Gram convergence check: random 256x256 batch (cfg5 shape) with
CS_GRAM_CHECK=2 (check after every rotating sweep, verdict ignored) vs =0."""
import os
import subprocess
import sys

code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2506_05617_b200 import engine
dev = torch.device("cuda:0")
g = torch.Generator(device="cpu").manual_seed(1)
base = torch.randn(64, 256, 256, dtype=torch.complex64, generator=g)
N = 8192
blocks = base.to(dev).repeat(N // 64, 1, 1).contiguous()
for vec in (True,):
    best = 1e9
    for _ in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = engine.batched_svd(blocks, "f32", vec); e1.record()
        torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
    print(vec, best, out.info.float().mean().item(), engine.plan_kind(N, 256, 256, "f32", vec), flush=True)
'''
res = {}
for mode in ("0", "2"):
    env = dict(os.environ, CS_GRAM_CHECK=mode)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    print(out.stderr[-2000:]) if out.returncode else None
    for line in out.stdout.splitlines():
        vec, t, sw, *_ = line.split()
        res[(mode, vec)] = (float(t), float(sw))
for vec in ("True",):
    t0, sw = res[("0", vec)]
    t2, _ = res[("2", vec)]
    checks = sw - 1  # one check after every rotating sweep
    print(f"vectors={vec}: per sweep {t0 / sw:.1f} ms, per Gram check {(t2 - t0) / checks:.2f} ms "
          f"({(t2 - t0) / checks / (t0 / sw) * 100:.1f}% of a sweep)")
