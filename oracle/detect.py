"""Oracle: detection, threshold, union and coefficient resolve of one round
(test infrastructure only, see oracle/__init__.py).

Alg. 1:
  Step 1 & 2a: per node g, keep k_t whose coefficient "is among the largest
      s_local (in absolute value) ... and |p~| >= theta"; union over g and rounds i.
  Step 2d: per node g, Algorithm A gives the <= s~ largest coefficients, each >= theta.
  Step 2e: I^(1..t) := I^(1..t) cup J~_{t,i,g}  (union over g, gray modification).

Readings:
  Z1  Algorithm A = L random R1Ls sharing M.  Detection key of candidate k at node g is
      kappa_min(k,g) = min_l kappa_l,  kappa_l = fl(fl(re*re) + fl(im*im)) of v_l(k,g).
      Values are resolved after the union from the lowest lattice where k is alias-free with
      respect to the node's own detected set D_g; fallback: componentwise median over l.
  Z5  theta relative to the round's max magnitude: kappa >= theta^2 with
      theta^2 = fl(fl(theta_rel*theta_rel) * kappa_max); absolute theta^2 = fl(theta_abs^2).
      Exact zeros are never detected (kappa > 0, as with the paper's theta > 0).
  Z6  top-s~ order: kappa desc, candidate index asc.     Z7  fewer than s~ pass: keep all.
  Z24 "aggregated over all mesh nodes": votes_k = sum_g [k in D_g]; I_round = {votes >= 1}.
  Z25 fragile decisions: a key >= theta - eps within eps = 1e-10 max m (m = sqrt(kappa_min)) of a
      different key on the other side of the node's s~-cut, or an in-cut key within eps of theta
      (two-sided; bit-equal keys and swaps below theta never).
"""
from __future__ import annotations

import numpy as np


def kappa(V: np.ndarray) -> np.ndarray:
    """fl(fl(re*re) + fl(im*im)) elementwise (numpy never contracts to FMA)."""
    re = np.real(V)
    im = np.imag(V)
    return re * re + im * im


def kappa_min(V: np.ndarray) -> np.ndarray:
    """Detection key [G][|J|] from per-lattice values V [L][G][|J|] (Z1)."""
    return kappa(V).min(axis=0)


def theta_squared(kmin: np.ndarray, theta_rel: float, theta_abs: float = 0.0) -> float:
    """theta^2 of the round (Z5; paper's absolute theta at P:278 when theta_abs > 0)."""
    if theta_abs > 0.0:
        return float(np.float64(theta_abs) * np.float64(theta_abs))
    kmax = np.float64(kmin.max()) if kmin.size else np.float64(0.0)
    return float(np.float64(np.float64(theta_rel) * np.float64(theta_rel)) * kmax)


def select(kmin: np.ndarray, s_tilde: int, theta2: float):
    """Per-node detected sets D_g (ascending candidate index) and votes."""
    G, nJ = kmin.shape
    idx = np.arange(nJ)
    D = []
    votes = np.zeros(nJ, dtype=np.int64)
    for g in range(G):
        order = np.lexsort((idx, -kmin[g]))                  # kappa desc, index asc (Z6)
        top = order[:s_tilde]
        keep = top[(kmin[g, top] >= theta2) & (kmin[g, top] > 0.0)]
        Dg = np.sort(keep)
        D.append(Dg)
        votes[Dg] += 1
    return D, votes


def resolve(V: np.ndarray, bins: np.ndarray, D: list, det: np.ndarray):
    """Coefficient of every k in det (this round's union) at every node g (Z1, a12).

    l*(k,g) = min { l : no k' in D_g \\ {k} has b_l(k') = b_l(k) }; c = v_{l*}(k,g);
    if no such l exists: componentwise (lower) median over l, lstar = -1.
    Returns (coef complex [G][n_det], lstar int [G][n_det]).
    """
    L, G, _ = V.shape
    nd = det.shape[0]
    M = int(bins.max()) + 1 if bins.size else 1
    coef = np.empty((G, nd), dtype=np.complex128)
    lstar = np.full((G, nd), -1, dtype=np.int64)
    for g in range(G):
        Dg = np.asarray(D[g], dtype=np.int64)
        own = np.isin(det, Dg).astype(np.int64)          # is k itself a member of D_g
        free = np.zeros((L, nd), dtype=bool)
        for l in range(L):
            # number of members of D_g in each bin of lattice l
            cnt = np.bincount(bins[l, Dg], minlength=M) if Dg.size else np.zeros(M, np.int64)
            free[l] = (cnt[bins[l, det]] - own) == 0      # no *other* member shares k's bin
        for q in range(nd):
            k = int(det[q])
            hit = np.nonzero(free[:, q])[0]
            if hit.size:
                coef[g, q] = V[hit[0], g, k]
                lstar[g, q] = hit[0]
            else:
                re = np.sort(np.real(V[:, g, k]))[(L - 1) // 2]
                im = np.sort(np.imag(V[:, g, k]))[(L - 1) // 2]
                coef[g, q] = re + 1j * im
    return coef, lstar


def fragile(kmin: np.ndarray, s_tilde: int, theta2: float, band: float = 1e-10) -> np.ndarray:
    """Boolean [G][|J|]: decisions a perturbation of the keys within the Z25 band could flip.

    With m = sqrt(kappa_min), eps = band * max m and node g's candidates in the selection order
    (m desc, index asc; Z6), the first s~ of that order are "in", the rest "out".
    (k, g) is fragile when
      * m >= theta - eps and an "in" k has an "out" k' with m' != m and m' >= m - eps (the two
        could swap), or an "out" k has an "in" k' with m' != m and m' <= m + eps;
      * or k is "in" and |m - theta| <= eps (the threshold decision, Z5).
    A swap of two keys below theta - eps changes no D_g (neither is detected either way), and
    bit-equal keys (e.g. two candidates in one bin of the minimising lattice) are ordered by
    index on both sides, so neither makes a decision fragile."""
    m = np.sqrt(kmin)
    G, nJ = kmin.shape
    eps = band * (m.max() if m.size else 0.0)
    theta = np.sqrt(theta2)
    s = min(s_tilde, nJ)
    idx = np.arange(nJ)
    out = np.zeros_like(kmin, dtype=bool)
    for g in range(G):
        # order and equality on the key kappa itself (two keys 1 ulp apart can share one sqrt);
        # distances on m
        order = np.lexsort((idx, -kmin[g]))
        kv = kmin[g][order]
        mv = m[g][order]
        ksel, krest, msel, mrest = kv[:s], kv[s:], mv[:s], mv[s:]
        fr = np.zeros(nJ, dtype=bool)
        if krest.size and ksel.size:
            # in: the largest out-key strictly below (rest is descending)
            pos = np.searchsorted(-krest, -ksel, side="right")
            below = np.where(pos < krest.size, mrest[np.minimum(pos, krest.size - 1)], -np.inf)
            fr[:s] = below >= msel - eps
            # out: the smallest in-key strictly above (sel is descending)
            q = np.searchsorted(-ksel, -krest, side="left") - 1
            above = np.where(q >= 0, msel[np.maximum(q, 0)], np.inf)
            fr[s:] = above <= mrest + eps
        fr &= mv >= theta - eps
        fr[:s] |= np.abs(msel - theta) <= eps
        out[g, order] = fr
    return out


def detect_round(V: np.ndarray, bins: np.ndarray, s_tilde: int, theta_rel: float,
                 theta_abs: float = 0.0, want_coef: bool = True) -> dict:
    """One round's a8-a12: keys, threshold, per-g select, votes, union, resolve."""
    kmin = kappa_min(V)
    th2 = theta_squared(kmin, theta_rel, theta_abs)
    D, votes = select(kmin, s_tilde, th2)
    det = np.nonzero(votes > 0)[0]
    out = dict(kappa_min=kmin, theta2=th2, D=D, votes=votes, det=det)
    if want_coef:
        out["coef"], out["lstar"] = resolve(V, bins, D, det)
    return out
