"""Quick check of the tensor-core blocked kernel on a cfg5 sub-range:
sigma vs the scalar panel kernel (CS_TCB=0 run in a subprocess), sweeps,
factor orthonormality, and the SVD-phase time.  python tools/tcb_check.py [COUNT] [WARM]"""
import json, os, subprocess, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05617_b200 import configs, engine  # noqa: E402
from paper_2506_05617_b200.pipeline import lfa_device  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 64
warm = sys.argv[2] != "0" if len(sys.argv) > 2 else True
dev = torch.device("cuda:0")
layer = configs.WORKLOADS[5].layers[0]
wd = torch.from_numpy(configs.layer_weights(layer)).to(dev)
tm = engine.Timer(dev)
res = lfa_device(wd, layer.n, layer.m, "f32", True, u0=0, count=count, timer=tm, warm_start=warm, assemble=False)
torch.cuda.synchronize()
t_svd = tm.seconds("t1", "t2")
tm = engine.Timer(dev)
res = lfa_device(wd, layer.n, layer.m, "f32", True, u0=0, count=count, timer=tm, warm_start=warm, assemble=False)
torch.cuda.synchronize()
t_svd = min(t_svd, tm.seconds("t1", "t2"))
sig = res.sigma.cpu().numpy()
info = res.info.cpu().numpy()
Aall = engine.symbol_field(wd, layer.n, layer.m, "f32", half=True, f_first=0, f_count=count)
fro = (Aall.abs().double() ** 2).sum(dim=(1, 2)).cpu().numpy()
del Aall
en = (np.sum(sig.astype(np.float64) ** 2, axis=1) - fro) / fro
out = {"count": count, "warm": warm, "tcb": os.environ.get("CS_TCB", "1"), "svd_ms": 1e3 * t_svd,
       "energy_bias": float(en.mean()), "energy_maxabs": float(np.abs(en).max()),
       "sweeps_mean": float(info.mean()), "sweeps_max": int(info.max()), "failed": int((info <= 0).sum())}
U = res.U[: min(count, 8)].cpu().numpy().astype(np.complex128)
V = res.V[: min(count, 8)].cpu().numpy().astype(np.complex128)
A = engine.symbol_field(wd, layer.n, layer.m, "f32", half=True, f_first=0, f_count=min(count, 8)).cpu().numpy().astype(np.complex128)
out["orthU"] = float(max(np.abs(u.conj().T @ u - np.eye(u.shape[1])).max() for u in U))
out["orthV"] = float(max(np.abs(v.conj().T @ v - np.eye(v.shape[1])).max() for v in V))
out["recon"] = float(max(np.abs((U[i] * sig[i]) @ V[i].conj().T - A[i]).max() / sig[i, 0] for i in range(len(U))))
r64 = lfa_device(wd, layer.n, layer.m, "f64", True, u0=0, count=count, warm_start=warm, assemble=False)
s64 = r64.sigma.cpu().numpy()
out["max_rel_vs_f64"] = float((np.abs(sig - s64).max(axis=1) / s64[:, 0]).max())
out["mean_rel_vs_f64"] = float((np.abs(sig - s64).max(axis=1) / s64[:, 0]).mean())
del r64
if os.environ.get("CS_TCB", "1") != "0" and not os.environ.get("CS_NO_SCALAR"):
    np.save("/tmp/sig_tcb.npy", sig)
    env = dict(os.environ, CS_TCB="0")
    subprocess.run([sys.executable, __file__, str(count), "1" if warm else "0"], env=env, check=True)
    ref = np.load("/tmp/sig_ref.npy")
    out["max_rel_vs_scalar"] = float((np.abs(sig - ref).max(axis=1) / ref[:, 0]).max())
else:
    np.save("/tmp/sig_ref.npy", sig)
print(json.dumps(out), flush=True)
