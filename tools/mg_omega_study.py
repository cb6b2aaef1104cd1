"""CPU study: CG iterations of the multigrid-preconditioned CG for per-level damped-Jacobi weights
(fine level, level 1, level 2, levels >= 3), V(1,1), bilinear P, rediscretised coarse operators:

    python tools/mg_omega_study.py CONFIG SAMPLES [scan]

Result (configs 1-5): (0.8, 1, 1, 1) never needs more iterations than (0.8, 0.8, 0.8, 0.8) and
saves one at configs 3-5 (config 5: 14 -> 13, relative residual after 12 iterations 3.2e-11 ->
3.8e-12); fine weights 0.75 / 0.85 cost one or two iterations; averaging the coefficient over the
coarse triangles instead of sampling its centroid changes nothing on these fields."""
import itertools, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/tools")
from mg_smoother_study import stiffness, prolong
from oracle import fe
from usfft_inputs import config


def build(n, model, y, nlev):
    As, Ps, m = [], [], n
    for l in range(nlev):
        As.append(stiffness(m, model, y).tocsr())
        if l < nlev - 1: Ps.append(prolong(m // 2).tocsr())
        m //= 2
    return As, Ps, np.linalg.inv(As[-1].toarray())


def vc(l, r, As, Ps, Ainv, w):
    if l == len(As) - 1: return Ainv @ r
    A, P, D, om = As[l], Ps[l], As[l].diagonal(), w[min(l, len(w) - 1)]
    x = om * r / D
    x = x + P @ vc(l + 1, P.T @ (r - A @ x), As, Ps, Ainv, w)
    return x + om * (r - A @ x) / D


def pcg(A, b, M, tol=1e-12, maxit=60):
    x = np.zeros_like(b); r = b.copy(); z = M(r); p = z.copy(); rz = r @ z; bb = b @ b
    hist = []
    for it in range(1, maxit + 1):
        q = A @ p; alpha = rz / (p @ q); x += alpha * p; r -= alpha * q
        hist.append(np.sqrt(r @ r / bb))
        if r @ r <= tol * tol * bb: return it, hist
        z = M(r); rz2 = r @ z; p = z + (rz2 / rz) * p; rz = rz2
    return maxit, hist


if __name__ == "__main__":
    cfgk, ns = int(sys.argv[1]), int(sys.argv[2])
    model = config(cfgk); n = model["n"]; nlev = int(np.log2(n)) - 1
    ws = [(0.8, 0.8, 0.8, 0.8), (0.8, 1.0, 1.0, 1.0), (0.8, 0.9, 0.9, 0.9), (0.75, 1.0, 1.0, 1.0), (0.85, 1.0, 1.0, 1.0)]
    if len(sys.argv) > 3:
        ws = list(itertools.product([0.78, 0.8, 0.82], [0.9, 1.0, 1.1], [0.9, 1.0, 1.1], [0.9, 1.0, 1.1]))
    res = {}
    for y in np.random.default_rng(2).random((ns, model["d"])):
        As, Ps, Ainv = build(n, model, y, nlev)
        cx, cy = fe.centroids(n)
        _, b = fe.assemble(n, np.ones_like(cx), fe.f_values(model, cx, cy))
        for w in ws:
            res.setdefault(w, []).append(pcg(As[0], b, lambda r: vc(0, r, As, Ps, Ainv, w)))
    for w, v in sorted(res.items(), key=lambda kv: np.mean([it for it, _ in kv[1]])):
        print(cfgk, w, "iterations", [it for it, _ in v],
              "relres before the last %.1e" % np.exp(np.mean(np.log([h[-2] for _, h in v]))))
