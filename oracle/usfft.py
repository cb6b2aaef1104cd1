"""Oracle: Algorithm 1 "The usFFT on a set T_G" step by step (test infrastructure only).

Follows Alg. 1 in the paper's order and notation, with Algorithm A realised as
described in oracle/detect.py (Z1) and the round plan of oracle/plan.py (Z2-Z4):

  Step 1 & 2a: for t = 1..d, i = 1..r: line nodes, one black-box call for all G
      nodes, per-node length-K_t DFT, per-node top-s_local >= theta, union over g and i.
      An empty I^(t) becomes {0} (Z9).
  Step 2: for t = 2..d: (r~, s~) = (r, s_local) if t < d else (1, s);
      for i = 1..r~: x'_{t+1..d}, sampling set for J_t = I^(1..t-1) x I^(t),
      samples for every chi_g, Algorithm A per g, union.
  Output (Z16): I = I^(1..d) and the coefficients resolved in the final round (t = d, r~ = 1).
"""
from __future__ import annotations

import numpy as np

from . import detect, dft, lattice, plan


def mode_r_lattice(J: np.ndarray, seed: int, t: int, i: int, N: int):
    """Single reconstructing R1L for J (mode R, Z2)."""
    M = plan.next_lattice_prime(max(2 * J.shape[0], N + 1))
    while M <= plan.MODE_R_MAX_M:
        for trial in range(plan.MODE_R_TRIES):
            z = plan.mode_r_z(seed, t, i, M, trial)
            if lattice.injective(lattice.bins(J, [z], M)[0]):
                return M, [z]
        M = plan.next_lattice_prime(M + 1)
    raise RuntimeError("no reconstructing lattice below the M cap")


def round_plan(cfg: dict, t: int, i: int, nJ: int, s_tilde: int, J=None):
    """(M, L, z) of a Step-2 round (Z2)."""
    if cfg.get("mode", "A") == "R":
        M, z = mode_r_lattice(J, cfg["seed"], t, i, cfg["N"])
        return M, 1, z
    # optional lattice factor f (Step-2 lattices sized for f s~, the Z2 rule at f s~)
    M = plan.lattice_size(s_tilde * int(cfg.get("lattice_factor", 1)), cfg["N"])
    L = plan.num_lattices(nJ)
    return M, L, plan.z_vectors(cfg["seed"], t, i, M, L)


def run(cfg: dict, blackbox, log: list | None = None, trace: list | None = None) -> dict:
    """Whole Alg. 1 detection (Steps 1-2) on a black box Y [d][B] -> samples [G][B].

    cfg keys: d, N, s, s_local, r, seed, theta_rel, theta_abs, mode ('A' or 'R').
    trace: if a list, every Step-2 round's detect_round() dict is appended (with its bins).
    """
    d, N = cfg["d"], cfg["N"]
    s, s_local, r, seed = cfg["s"], cfg["s_local"], cfg["r"], cfg["seed"]
    th_rel, th_abs = cfg.get("theta_rel", 1e-6), cfg.get("theta_abs", 0.0)
    K = 2 * N + 1
    kt_full = np.arange(-N, N + 1, dtype=np.int64)
    n_samples = 0

    # ---- Step 1 & 2a: single frequency component identification --------------------------
    I1d = []
    for t in range(1, d + 1):
        found = np.zeros(K, dtype=bool)
        J = kt_full.reshape(-1, 1)
        bins = lattice.bins(J, [[1]], K)                                 # k_t mod K_t
        for i in range(1, r + 1):
            xs = plan.shift(seed, 1, t, i, d)
            Y = lattice.nodes(K, [[1]], xs, 1, line_axis=t - 1)
            U = blackbox(Y)
            n_samples += Y.shape[1]
            V = dft.round_values(U, K, 1, bins)
            res = detect.detect_round(V, bins, s_local, th_rel, th_abs, want_coef=False)
            found[res["det"]] = True
            if log is not None:
                log.append(dict(step=1, t=t, i=i, B=Y.shape[1], nJ=K, n_det=len(res["det"]),
                                theta2=res["theta2"]))
        It = kt_full[found]
        I1d.append(It if It.size else np.zeros(1, dtype=np.int64))      # Z9

    # ---- Step 2: coupling frequency components identification -----------------------------
    I_prev = I1d[0].reshape(-1, 1)
    coef = None
    for t in range(2, d + 1):
        r_t, s_t = (r, s_local) if t < d else (1, s)
        J = lattice.candidates(I_prev, I1d[t - 1])
        found = np.zeros(J.shape[0], dtype=bool)
        for i in range(1, r_t + 1):
            M, L, z = round_plan(cfg, t, i, J.shape[0], s_t, J)
            xs = plan.shift(seed, 2, t, i, d)
            Y = lattice.nodes(M, z, xs, t)
            U = blackbox(Y)
            n_samples += Y.shape[1]
            bins = lattice.bins(J, z, M)
            V = dft.round_values(U, M, L, bins)
            res = detect.detect_round(V, bins, s_t, th_rel, th_abs, want_coef=(t == d))
            found[res["det"]] = True
            if trace is not None:
                res["bins"] = bins
                trace.append(res)
            if t == d:
                coef = res["coef"]
            if log is not None:
                log.append(dict(step=2, t=t, i=i, M=M, L=L, B=Y.shape[1], nJ=J.shape[0],
                                n_det=len(res["det"]), theta2=res["theta2"]))
        I_prev = J[found]
        if I_prev.shape[0] == 0:
            return dict(I=I_prev, C=np.zeros((0, 0), complex), n_samples=n_samples, I1d=I1d)
    return dict(I=I_prev, C=coef, n_samples=n_samples, I1d=I1d)
