"""Warm start by extrapolation on the unitary group (study, numpy complex128):
first-order X' = A_f V_p versus second-order X'' = A_f V_p (V_gp^H V_p) along a
lattice chain gp -> p -> f of the cfg5 layer; reports the off-diagonal mass of
X^H X and the sweeps of the K2 / K3 numpy models (tools/blocksim.py rules).
python tools/extrap_study.py I0 J0 [DIR]"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = [sys.argv[0]] + sys.argv[1:]
i0 = int(sys.argv[1]) if len(sys.argv) > 1 else 5
j0 = int(sys.argv[2]) if len(sys.argv) > 2 else 7
dirn = sys.argv[3] if len(sys.argv) > 3 else "i"
sims = sys.argv[4] if len(sys.argv) > 4 else "k3"
from paper_2506_05617_b200 import configs  # noqa: E402
import importlib.util
spec = importlib.util.spec_from_file_location("bs", os.path.join(os.path.dirname(__file__), "blocksim_lib.py"))
bs = importlib.util.module_from_spec(spec); spec.loader.exec_module(bs)
layer = configs.WORKLOADS[5].layers[0]
w = configs.layer_weights(layer).astype(np.float64)
co, ci, kh, kw = w.shape
n, m = layer.n, layer.m
def sym(i, j):
    t1, t2 = 2 * np.pi * i / n, 2 * np.pi * j / m
    ph = np.exp(1j * (t1 * np.arange(kh)[:, None] + t2 * np.arange(kw)[None, :]))
    return np.einsum("oipq,pq->oi", w, ph)
pts = [(i0 + (k if dirn == "i" else 0), j0 + (k if dirn == "j" else 0)) for k in range(3)]
A = [sym(*p) for p in pts]
V = []
for a in A[:2]:
    _, s, vh = np.linalg.svd(a)
    V.append(vh.conj().T)
def off(X):
    G = X.conj().T @ X
    d = np.sqrt(np.abs(np.diag(G)).real)
    Gn = G / d[:, None] / d[None, :]
    np.fill_diagonal(Gn, 0)
    return np.abs(Gn).max(), np.linalg.norm(Gn) / np.sqrt(G.shape[0])
X1 = A[2] @ V[1]
M = V[0].conj().T @ V[1]
X2 = A[2] @ (V[1] @ M)
print(pts, "first-order off max/rms %.3e %.3e" % off(X1), " extrapolated %.3e %.3e" % off(X2), flush=True)
tol = 5e-6
for name, X in (("first", X1), ("extrap", X2)):
    if "k2" in sims:
        sw, _ = bs.k2(X, tol); print(f"  {name}: K2 sweeps {sw}", flush=True)
    if "k3" in sims:
        sw, _ = bs.k3(X, tol); print(f"  {name}: K3 sweeps {sw}", flush=True)
