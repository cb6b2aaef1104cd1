"""Oracle: rank-1 lattice nodes and candidate index maps (test infrastructure only).

* R1L: Lambda(z, M) = { (i/M) z mod 1 : i = 0..M-1 }                    (Sec. 2.2)
* node components  y~_{i,j} = (i/M) z_j mod 1                            (eq. lattice_nodes)
* Step 2b sampling set X_{t,i} = {(x~, x'_{t+1}, .., x'_d) : x~ in X}   (Alg. 1 Step 2b)
* Step 1 & 2a line nodes x^(l)_j = l/K_t (j = t), x'_j (j != t)          (Alg. 1)
* a frequency k is read from bin (k . z) mod M of the length-M DFT      (
  it follows from e^{2 pi i k.y_i} = e^{2 pi i i (k.z)/M})

Layouts (shared with the boundary): nodes are [d][B] with sample b = l*M + i
fastest; candidate j = a*n1 + b for a over the rows of I_prev and b over kt (Z10).
"""
from __future__ import annotations

import numpy as np


def nodes(M: int, z, shift, t: int, line_axis: int = -1) -> np.ndarray:
    """Sampling nodes of one round, fp64 [d][L*M].

    Step 2 (line_axis < 0): for lattice l and node i, component j (0-based) is
        ((i * z[l][j]) mod M) / M   for j < t   (lattice part x~ in T^t)
        shift[j]                    for j >= t  (shared trailing x')
    Step 1 (line_axis = t-1, z = [[1]], M = K_t): component line_axis is ((i*1) mod K)/K = i/K
     and every other component is shift[j].

    The division of the exact integer (i*z mod M) by M is one IEEE division.
    """
    z = np.asarray(z, dtype=np.int64).reshape(len(z), -1)
    L = z.shape[0]
    d = len(shift)
    i = np.arange(M, dtype=np.int64)
    y = np.empty((d, L * M), dtype=np.float64)
    for j in range(d):
        y[j, :] = shift[j]
    for l in range(L):
        cols = slice(l * M, (l + 1) * M)
        if line_axis >= 0:
            y[line_axis, cols] = ((i * z[l, 0]) % M).astype(np.float64) / float(M)
        else:
            for j in range(t):
                y[j, cols] = ((i * z[l, j]) % M).astype(np.float64) / float(M)
    return y


def candidates(I_prev, kt) -> np.ndarray:
    """J_t = I^(1..t-1) x I^(t) as int rows [|J|][t] in candidate order j = a*n1 + b (Z10).

    P:310: J_t := (I^(1,..,t-1) x I^(t)) cap P_(1..t)(Gamma); for a box Gamma the cap is
    automatic because every factor already lies in the box.
    """
    I_prev = np.asarray(I_prev, dtype=np.int64).reshape(len(I_prev), -1)
    kt = np.asarray(kt, dtype=np.int64).reshape(-1)
    n_prev, n1 = I_prev.shape[0], kt.shape[0]
    left = np.repeat(I_prev, n1, axis=0)                 # row a repeated for every b
    right = np.tile(kt, n_prev).reshape(-1, 1)           # b runs fastest
    return np.concatenate([left, right], axis=1)


def bins(J, z, M: int) -> np.ndarray:
    """Index map b_l(k) = (k . z_l) mod M in [0, M) for every candidate k in J, int [L][|J|].

    S:119-127 (residues), S:158 (read bin k.z mod M).  Exact int64 arithmetic: |k_j| <= 2^15,
    z < 2^26, t <= 64 keeps every partial sum below 2^47.
    """
    J = np.asarray(J, dtype=np.int64)
    z = np.asarray(z, dtype=np.int64).reshape(-1, J.shape[1])
    return np.mod(z @ J.T, M)      # numpy mod of int64 by positive M lies in [0, M)


def injective(bins_row) -> bool:
    """Reconstructing property of a single R1L for J: the map k -> k.z mod M is one-to-one
    (single R1L approach, Table 1 row 1 P:242)."""
    seen = set()
    for b in bins_row:
        b = int(b)
        if b in seen:
            return False
        seen.add(b)
    return True
