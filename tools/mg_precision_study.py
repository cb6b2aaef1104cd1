"""CPU study (numpy/scipy): CG iterations of the multigrid-preconditioned CG with the V-cycle in
fp64 vs fp32 (from level 1, or from the fine level): python tools/mg_precision_study.py CONFIG SAMPLES"""
import sys, numpy as np, scipy.sparse as sp
ROOT = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tools")
from mg_smoother_study import stiffness, prolong
from oracle import fe
from usfft_inputs import config

def build(n, model, y, nlev):
    As, Ps = [], []
    m = n
    for l in range(nlev):
        As.append(stiffness(m, model, y).tocsr())
        if l < nlev - 1: Ps.append(prolong(m // 2).tocsr())
        m //= 2
    return As, Ps, np.linalg.inv(As[-1].toarray())

def vc(l, r, As, Ps, Ainv, dt, lev32, om=0.8):
    if l == len(As) - 1:
        return (Ainv @ r.astype(np.float64)).astype(r.dtype)
    A = As[l]; P = Ps[l]
    if l >= lev32:
        A = A.astype(np.float32); P = P.astype(np.float32); r = r.astype(np.float32)
    D = A.diagonal()
    x = om * r / D
    rc = P.T @ (r - A @ x)
    x = x + P @ vc(l + 1, rc, As, Ps, Ainv, dt, lev32, om)
    x = x + om * (r - A @ x) / D
    return x

def pcg(A, b, M, tol=1e-12, maxit=200):
    x = np.zeros_like(b); r = b.copy(); z = M(r).astype(np.float64); p = z.copy(); rz = r @ z; bb = b @ b
    for it in range(1, maxit + 1):
        q = A @ p; alpha = rz / (p @ q); x += alpha * p; r -= alpha * q
        if r @ r <= tol * tol * bb: return it, x
        z = M(r).astype(np.float64); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return maxit, x

cfgk = int(sys.argv[1]); ns = int(sys.argv[2])
model = config(cfgk); n = model["n"]; nlev = int(np.log2(n)) - 1
rng = np.random.default_rng(0)
res = {}
for y in rng.random((ns, model["d"])):
    As, Ps, Ainv = build(n, model, y, nlev)
    cx, cy = fe.centroids(n)
    _, b = fe.assemble(n, np.ones_like(cx), fe.f_values(model, cx, cy))
    xs = None
    for lev32 in (99, 1, 0):
        it, x = pcg(As[0], b, lambda r: vc(0, r, As, Ps, Ainv, None, lev32))
        if xs is None: xs = x
        res.setdefault(lev32, []).append((it, np.abs(x - xs).max() / np.abs(xs).max()))
for k, v in res.items():
    print("fp32 from level", k, "iters", [a for a, _ in v], "maxdiff", max(b for _, b in v))
