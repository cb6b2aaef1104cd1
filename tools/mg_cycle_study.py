"""CPU study: CG iterations of the multigrid-preconditioned CG for V(1,1) / V(2,2) cycles and
smoother weights on a config: python tools/mg_cycle_study.py CONFIG SAMPLES"""
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

def vc(l, r, As, Ps, Ainv, nu, om, gam=1):
    if l == len(As) - 1:
        return Ainv @ r
    A = As[l]; P = Ps[l]; D = A.diagonal()
    k = nu(l)
    x = om * r / D
    for _ in range(k - 1): x = x + om * (r - A @ x) / D
    for _ in range(gam):
        rc = P.T @ (r - A @ x)
        x = x + P @ vc(l + 1, rc, As, Ps, Ainv, nu, om, 1)
    for _ in range(k): x = x + om * (r - A @ x) / D
    return x

def pcg(A, b, M, tol=1e-12, maxit=200):
    x = np.zeros_like(b); r = b.copy(); z = M(r); p = z.copy(); rz = r @ z; bb = b @ b
    for it in range(1, maxit + 1):
        q = A @ p; alpha = rz / (p @ q); x += alpha * p; r -= alpha * q
        if r @ r <= tol * tol * bb: return it
        z = M(r); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return maxit

cfgk = int(sys.argv[1]); ns = int(sys.argv[2])
model = config(cfgk); n = model["n"]; nlev = int(np.log2(n)) - 1
rng = np.random.default_rng(0)
variants = {"V11 w.8": (lambda l: 1, 0.8), "V11 w.7": (lambda l: 1, 0.7), "V11 w.9": (lambda l: 1, 0.9),
            "V22 all": (lambda l: 2, 0.8), "V22 fine": (lambda l: 2 if l == 0 else 1, 0.8),
            "V21fine+L1": (lambda l: 2 if l <= 1 else 1, 0.8), "V11 coarse2": (lambda l: 1 if l <= 1 else 2, 0.8)}
res = {k: [] for k in variants}
for y in rng.random((ns, model["d"])):
    As, Ps, Ainv = build(n, model, y, nlev)
    cx, cy = fe.centroids(n)
    _, b = fe.assemble(n, np.ones_like(cx), fe.f_values(model, cx, cy))
    for k, (nu, om) in variants.items():
        res[k].append(pcg(As[0], b, lambda r: vc(0, r, As, Ps, Ainv, nu, om)))
for k, v in res.items(): print(f"{k:12s} {np.mean(v):.2f} {v}")
