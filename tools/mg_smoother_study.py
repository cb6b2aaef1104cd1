"""CPU study (numpy/scipy): CG iterations of the multigrid-preconditioned CG of k_pcg_mg for
different smoothers, on config-2 samples.  Levels n, n/2, n/4 smoothed, n/8 exact; bilinear P,
R = P^T, rediscretised coarse operators (coefficients at the coarse centroids).

    python tools/mg_smoother_study.py [--samples 20]
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def stiffness(n, model, y):
    from oracle import fe
    cx, cy = fe.centroids(n)
    a = fe.coefficient(model, y, cx, cy)
    ab, _ = fe.assemble(n, a, np.zeros_like(cx))
    return sp.csr_matrix(fe.banded_to_dense(ab))


def prolong(nc):
    """bilinear P from the (nc-1)^2 interior nodes of the coarse mesh to the (2nc-1)^2 fine ones."""
    nf = 2 * nc
    rows, cols, vals = [], [], []
    idx_c = lambda I, J: (J - 1) * (nc - 1) + (I - 1)
    for j in range(1, nf):
        for i in range(1, nf):
            r = (j - 1) * (nf - 1) + (i - 1)
            I0, J0 = i // 2, j // 2
            wi = [(I0, 1.0)] if i % 2 == 0 else [(I0, 0.5), (I0 + 1, 0.5)]
            wj = [(J0, 1.0)] if j % 2 == 0 else [(J0, 0.5), (J0 + 1, 0.5)]
            for I, a in wi:
                for J, b in wj:
                    if 1 <= I <= nc - 1 and 1 <= J <= nc - 1:
                        rows.append(r); cols.append(idx_c(I, J)); vals.append(a * b)
    return sp.csr_matrix((vals, (rows, cols)), shape=((nf - 1) ** 2, (nc - 1) ** 2))


def colors(n):
    jj, ii = np.meshgrid(np.arange(1, n), np.arange(1, n), indexing="ij")
    return ((ii + jj) % 2).reshape(-1)


def make_smoother(kind, A, n, omega):
    D = A.diagonal()
    col = colors(n)
    L = sp.tril(A, -1).tocsr()
    if kind == "jacobi":
        def pre(r, x):
            return x + omega * (r - A @ x) / D
        return pre, pre
    if kind == "jacobi2":
        def pre(r, x):
            for _ in range(2):
                x = x + omega * (r - A @ x) / D
            return x
        return pre, pre
    if kind == "rbgs":                       # red-black Gauss-Seidel: pre red->black, post black->red
        def sweep(r, x, c):
            m = col == c
            res = r - A @ x
            x = x.copy()
            x[m] += res[m] / D[m]
            return x

        def pre(r, x):
            return sweep(r, sweep(r, x, 0), 1)

        def post(r, x):
            return sweep(r, sweep(r, x, 1), 0)
        return pre, post
    raise ValueError(kind)


def build_levels(n, model, y, kind, omega, nlev=4):
    As, Ps, sm = [], [], []
    m = n
    for l in range(nlev):
        As.append(stiffness(m, model, y))
        if l < nlev - 1:
            Ps.append(prolong(m // 2))
            sm.append(make_smoother(kind, As[-1], m, omega))
        m //= 2
    Ainv = np.linalg.inv(As[-1].toarray())
    return As, Ps, sm, Ainv


def vcycle(l, r, As, Ps, sm, Ainv):
    if l == len(As) - 1:
        return Ainv @ r
    pre, post = sm[l]
    x = pre(r, np.zeros_like(r))
    rc = Ps[l].T @ (r - As[l] @ x)
    x = x + Ps[l] @ vcycle(l + 1, rc, As, Ps, sm, Ainv)
    return post(r, x)


def pcg_iters(A, b, M, tol=1e-12, maxit=200):
    x = np.zeros_like(b)
    r = b.copy()
    z = M(r)
    p = z.copy()
    rz = r @ z
    bb = b @ b
    for it in range(1, maxit + 1):
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        if r @ r <= tol * tol * bb:
            return it
        z = M(r)
        rz2 = r @ z
        p = z + (rz2 / rz) * p
        rz = rz2
    return maxit


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=12)
    ap.add_argument("--config", default="2")
    args = ap.parse_args()
    from oracle import fe
    from usfft_inputs import config
    key = int(args.config) if args.config.isdigit() else args.config
    model = config(key)
    if model["theta"] == "phi_delta":
        model["delta"] = fe.global_delta(401)
    n = model["n"]
    rng = np.random.default_rng(0)
    Ys = rng.random((args.samples, model["d"]))
    for kind, omega in (("jacobi", 0.8), ("jacobi", 0.7), ("jacobi", 0.9), ("jacobi2", 0.8), ("rbgs", 1.0)):
        its = []
        for y in Ys:
            As, Ps, sm, Ainv = build_levels(n, model, y, kind, omega)
            cx, cy = fe.centroids(n)
            _, b = fe.assemble(n, np.ones_like(cx), fe.f_values(model, cx, cy))
            its.append(pcg_iters(As[0], b, lambda r: vcycle(0, r, As, Ps, sm, Ainv)))
        print(f"{kind:8s} omega={omega}: iterations mean {np.mean(its):.2f} max {max(its)}", flush=True)


if __name__ == "__main__":
    main()
