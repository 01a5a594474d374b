"""Can the rotation-free check sweep be predicted?  (CPU study, numpy fp64.)

One-sided Jacobi with a circle (round-robin) parallel ordering on cfg5
symbol blocks, cold (V = I) and warm (V from the SVD of the neighbouring
frequency, as engine.warm_plan does).  Per sweep it prints the max ratio
r_k = |gamma|/sqrt(alpha beta) met during the sweep and the true residual
rho_k = max_{i<j} |x_i^H x_j|/(|x_i||x_j|) after it.

python tools/stopstudy.py [NFREQ]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as orc  # noqa: E402  (study tool, CPU)
from paper_2506_05617_b200 import configs  # noqa: E402

TOL = 5e-6


def rounds(n):
    pos = list(range(n))
    for _ in range(n - 1):
        yield np.array([pos[i] for i in range(n // 2)]), np.array([pos[n - 1 - i] for i in range(n // 2)])
        pos = [pos[0]] + [pos[-1]] + pos[1:-1]


def residual(X):
    nrm = np.linalg.norm(X, axis=0)
    G = (X.conj().T @ X) / np.outer(nrm, nrm)
    np.fill_diagonal(G, 0)
    return np.abs(G).max()


def jacobi(X, max_sweeps=20):
    out = []
    n = X.shape[1]
    for sw in range(max_sweeps):
        rmax = 0.0
        nrot = 0
        for a, b in rounds(n):
            x, y = X[:, a], X[:, b]
            al = np.sum(np.abs(x) ** 2, axis=0)
            be = np.sum(np.abs(y) ** 2, axis=0)
            ga = np.sum(x.conj() * y, axis=0)
            ag = np.abs(ga)
            ratio = ag / np.sqrt(al * be)
            rmax = max(rmax, ratio.max())
            act = ratio > TOL
            nrot += int(act.sum())
            if not act.any():
                continue
            agp = np.where(act, ag, 1.0)
            zeta = (be - al) / (2 * agp)
            t = np.sign(zeta + (zeta == 0)) / (np.abs(zeta) + np.sqrt(1 + zeta ** 2))
            c = 1 / np.sqrt(1 + t ** 2)
            s = c * t
            ph = np.where(act, ga / agp, 1.0)
            c = np.where(act, c, 1.0)
            s = np.where(act, s, 0.0)
            newx = c * x - s * np.conj(ph) * y
            newy = s * ph * x + c * y
            X[:, a], X[:, b] = newx, newy
        rho = residual(X)
        out.append((rmax, rho, nrot))
        if nrot == 0:
            break
    return out


def main():
    nf = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    layer = configs.WORKLOADS[5].layers[0]
    w = configs.layer_weights(layer).astype(np.float64)
    grid = orc.grid_frequencies(layer.n, layer.m)
    rng = np.random.default_rng(3)
    for f in rng.integers(0, layer.n * layer.m - 1, nf):
        A, An = orc.symbol_field(w, freqs=grid[[f, f + 1]])
        _, _, Vh = np.linalg.svd(An)
        for name, X in (("cold", A.copy()), ("warm", A @ Vh.conj().T)):
            hist = jacobi(X)
            print(f"f={f} {name}: " + "  ".join(f"[{r:.1e}->{p:.1e} n{k}]" for r, p, k in hist),
                  flush=True)


if __name__ == "__main__":
    main()
