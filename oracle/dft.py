"""Oracle: the lattice DFT along the sample axis (test infrastructure only).

Alg. 1 Step 1 & 2a:  p~_{t,k_t,g} = (1/K_t) sum_{l=0}^{K_t-1} p(chi_g, x^(l)) e^{-2 pi i l k_t / K_t}.
Rank-1 lattice version (Z18): for lattice l of a round and candidate k with bin
b = k.z_l mod M,
    v_l(k, g) = (1/M) sum_{i=0}^{M-1} u(x_g, y_{l,i}) e^{-2 pi i * i * b / M}.
Written as the plain definition: the phase index (i*b) mod M is an exact integer, the
twiddle is cos/sin of 2 pi m / M in fp64, the sum is a dot product (matmul as one step).
"""
from __future__ import annotations

import numpy as np


def twiddles(M: int):
    m = np.arange(M, dtype=np.float64)
    ang = 2.0 * np.pi * m / M
    return np.cos(ang), np.sin(ang)


def lattice_dft(U: np.ndarray, M: int, bins_needed: np.ndarray) -> np.ndarray:
    """(1/M) sum_i U[..., i] e^{-2 pi i (i*b mod M)/M} for each b in bins_needed.

    U: [..., M] real or complex samples of one lattice in node order i = 0..M-1.
    Returns complex [..., len(bins_needed)].
    """
    U = np.asarray(U)
    bins_needed = np.asarray(bins_needed, dtype=np.int64).reshape(-1)
    c, s = twiddles(M)
    i = np.arange(M, dtype=np.int64)
    out = np.empty(U.shape[:-1] + (bins_needed.shape[0],), dtype=np.complex128)
    chunk = max(1, (1 << 22) // max(M, 1))
    for c0 in range(0, bins_needed.shape[0], chunk):
        bsel = bins_needed[c0:c0 + chunk]
        m = (i[:, None] * bsel[None, :]) % M                       # exact phase index
        E = c[m] - 1j * s[m]                                        # e^{-2 pi i m / M}
        out[..., c0:c0 + chunk] = (U @ E) / M
    return out


def round_values(U: np.ndarray, M: int, L: int, bins: np.ndarray) -> np.ndarray:
    """v_l(k, g) for every lattice l, node g and candidate k: complex [L][G][|J|].

    U: [G][L*M] samples (lattice l occupies columns l*M .. l*M+M-1); bins: [L][|J|].
    Only the distinct bins in use are transformed (same values as the full spectrum).
    """
    U = np.asarray(U)
    G = U.shape[0]
    nJ = bins.shape[1]
    V = np.empty((L, G, nJ), dtype=np.complex128)
    for l in range(L):
        ub, inv = np.unique(bins[l], return_inverse=True)
        vals = lattice_dft(U[:, l * M:(l + 1) * M], M, ub)          # [G][n_unique]
        V[l] = vals[:, inv.reshape(-1)]
    return V
