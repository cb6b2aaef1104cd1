"""CPU study: CG iterations when the bottom V-cycle levels use the constant-coefficient operator
(a per-launch instead of per-sample K map): python tools/mg_constk_study.py CONFIG SAMPLES"""
import sys, numpy as np
ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tools")
from mg_smoother_study import stiffness, prolong
from oracle import fe
from usfft_inputs import config

def build(n, model, y, nlev, const_from):
    As, Ps = [], []
    m = n; l = 0
    while l < nlev:
        yy = y if l < const_from else np.full_like(y, 0.0)   # y = 0 -> sin map gives a = 1
        As.append(stiffness(m, model, yy).tocsr())
        if l < nlev - 1: Ps.append(prolong(m // 2).tocsr())
        m //= 2; l += 1
    return As, Ps, np.linalg.inv(As[-1].toarray())

def vc(l, r, As, Ps, Ainv, om=0.8):
    if l == len(As) - 1: return Ainv @ r
    A = As[l]; P = Ps[l]; D = A.diagonal()
    x = om * r / D
    x = x + P @ vc(l + 1, P.T @ (r - A @ x), As, Ps, Ainv, om)
    return x + om * (r - A @ x) / D

def pcg(A, b, M, tol=1e-12, maxit=200):
    x = np.zeros_like(b); r = b.copy(); z = M(r); p = z.copy(); rz = r @ z; bb = b @ b
    for it in range(1, maxit + 1):
        q = A @ p; alpha = rz / (p @ q); x += alpha * p; r -= alpha * q
        if r @ r <= tol * tol * bb: return it
        z = M(r); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return maxit

cfgk = int(sys.argv[1]); ns = int(sys.argv[2])
model = config(cfgk); n = model["n"]; nlev = int(np.log2(n)) - 1
rng = np.random.default_rng(1)
for y in rng.random((ns, model["d"])):
    cx, cy = fe.centroids(n)
    _, b = fe.assemble(n, np.ones_like(cx), fe.f_values(model, cx, cy))
    res = []
    for cf in (99, nlev - 2, nlev - 3):
        As, Ps, Ainv = build(n, model, y, nlev, cf)
        res.append(pcg(As[0], b, lambda r: vc(0, r, As, Ps, Ainv)))
    print("exact coarse", res[0], "| const bottom 2 levels", res[1], "| const bottom 3", res[2])
