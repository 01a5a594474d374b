# numpy model of K3 combination rules (K3 "Two combination passes"): python tools/blocksim.py SEED EPS [k2|k3|all]
"""Sweep counts of blocked one-sided Jacobi variants on warm-started blocks (numpy, complex128).
K3: per super-round, G = P^H P of the panel pair, all pair rotations from G at once,
combined as a product (small angles) or exp(E) (large); variants with a second pass."""
import numpy as np, sys
from scipy.linalg import expm

W = 16; NC = 256; C = NC // (2 * W)

def pair_cols(k, r, n):
    L = n - 1
    ca = 0 if k == 0 else ((k - 1 + r) % L) + 1
    cb = ((n - 2 - k + r) % L) + 1
    return ca, cb

def rot(al, be, g, tol):
    q = abs(g) ** 2
    if q <= tol * tol * al * be: return None
    ag = abs(g); d = be - al
    t = 2 * ag / (abs(d) + np.hypot(d, 2 * ag)); t = -t if d < 0 else t
    r = np.sqrt(1 + t * t); c = 1 / r; s = t / r
    return c, s * g / ag, (q > 0.05 ** 2 * al * be)

def superround(P, cols, full, tol, passes):
    idx = list(cols)
    Q = np.eye(2 * W, dtype=complex)
    rotated = False
    for _ in range(passes):
        G = (P[:, idx] @ Q).conj().T @ (P[:, idx] @ Q)
        prm = []; big = False
        nround = 2 * W - 1 if full else W
        for r in range(nround):
            for k in range(W):
                p, q = (pair_cols(k, r, 2 * W) if full else (k, W + (k + r) % W))
                R = rot(G[p, p].real, G[q, q].real, G[p, q], tol)
                if R: prm.append((p, q, R)); big |= R[2]
        if not prm: break
        rotated = True
        if not big:
            D = np.eye(2 * W, dtype=complex)
            for p, q, (c, w, _) in prm:
                J = np.eye(2 * W, dtype=complex); J[p, p] = c; J[q, q] = c; J[p, q] = w; J[q, p] = -np.conj(w)
                # column update convention: x' = c x - conj(w) y ... (a' = a c - b conj(w)), b' = a w + b c
                J = np.eye(2 * W, dtype=complex); J[p, p] = c; J[q, p] = -np.conj(w); J[p, q] = w; J[q, q] = c
                D = D @ J
            Qs = D
        else:
            E = np.zeros((2 * W, 2 * W), dtype=complex)
            for p, q, (c, w, _) in prm:
                s = abs(w); th = np.arctan2(s, c); f = th / s
                E[q, p] = -f * np.conj(w); E[p, q] = f * w
            Qs = expm(E)
        Q = Q @ Qs
    P[:, idx] = P[:, idx] @ Q
    return rotated

def k3(X, tol, passes=1, maxsw=40):
    P = X.copy()
    for sw in range(maxsw):
        any_rot = False
        for t in range(2 * C - 1):
            for c in range(C):
                a, b = pair_cols(c, t, 2 * C)
                cols = list(range(a * W, a * W + W)) + list(range(b * W, b * W + W))
                any_rot |= superround(P, cols, t == 0, tol, passes)
        if not any_rot: return sw + 1, P
    return -1, P

def k2(X, tol, maxsw=40):
    P = X.copy(); n = P.shape[1]
    for sw in range(maxsw):
        any_rot = False
        for r in range(n - 1):
            for k in range(n // 2):
                p, q = pair_cols(k, r, n)
                a, b = P[:, p], P[:, q]
                R = rot(np.vdot(a, a).real, np.vdot(b, b).real, np.vdot(a, b), tol)
                if R:
                    c, w, _ = R; any_rot = True
                    P[:, p], P[:, q] = a * c - b * np.conj(w), a * w + b * c
        if not any_rot: return sw + 1, P
    return -1, P

