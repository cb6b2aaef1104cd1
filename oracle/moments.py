"""Oracle: post-processing of the usFFT coefficients — expectation, variance and global
sensitivity indices (test infrastructure only, see oracle/__init__.py).

Expectation (Sec. 4.1 "Expectation value of the approximation"), per node x_g:
    E(u_{x_g}) = sum_{k in I} c_k D_k,   D_k = prod_j D_{k_j},
    periodic model (no periodization):   D_{k_j} = 1 if k_j = 0 else 0   (E = c_0);
    tent periodization (affine, eq. affine_ew):
        D_{k_j} = 2i / (pi k_j) for odd k_j, 1 for k_j = 0, 0 otherwise;
    phi_Delta periodization (lognormal):
        D_{k_j,Delta} = 2i / (pi k_j) e^{2 pi i k_j Delta} for odd k_j, 1 for k_j = 0, 0 otherwise.
Variance and GSI (eq. gsi, eq. J):
    sigma^2_g = sum_{k in I \\ {0}} |c_k|^2,
    rho(J_l) = sum_{k in J_l \\ {0}} |c_k|^2 / sigma^2_g,  J_l = {k in I : ||k||_0 = l};
rho is reported as 0 where sigma^2_g = 0 (reading Z30: the ratio is undefined there).
"""
from __future__ import annotations

import numpy as np

MAPS = ("sin", "tent", "phi_delta")


def d_factor(kind: str, kj: int, delta: float = 0.0) -> complex:
    """D_{k_j} of one component."""
    if kj == 0:
        return 1.0 + 0.0j
    if kind == "sin" or kj % 2 == 0:
        return 0.0j
    v = 2.0j / (np.pi * kj)
    if kind == "phi_delta":
        v = v * np.exp(2.0j * np.pi * kj * delta)
    return v


def d_weights(I: np.ndarray, kind: str, delta: float = 0.0) -> np.ndarray:
    """D_k = prod_j D_{k_j} for every row k of I [nI][d] -> complex [nI]."""
    I = np.asarray(I, dtype=np.int64)
    out = np.ones(I.shape[0], dtype=np.complex128)
    for a in range(I.shape[0]):
        for kj in I[a]:
            out[a] *= d_factor(kind, int(kj), delta)
    return out


def expectation(I: np.ndarray, C: np.ndarray, kind: str, delta: float = 0.0) -> np.ndarray:
    """E(u_{x_g}) = sum_k c_k D_k for every node: complex [G] (C is [G][nI])."""
    return np.asarray(C, dtype=np.complex128) @ d_weights(I, kind, delta)


def variance(I: np.ndarray, C: np.ndarray) -> np.ndarray:
    """sigma^2_g = sum_{k != 0} |c_k|^2: [G]."""
    nz = np.any(np.asarray(I) != 0, axis=1)
    A = np.abs(np.asarray(C)) ** 2
    return A[:, nz].sum(axis=1)


def gsi(I: np.ndarray, C: np.ndarray) -> np.ndarray:
    """rho(J_l) for l = 1..d: [G][d] (0 where sigma^2_g = 0)."""
    I = np.asarray(I)
    d = I.shape[1]
    ell = np.count_nonzero(I, axis=1)
    A = np.abs(np.asarray(C)) ** 2
    var = variance(I, C)
    out = np.zeros((A.shape[0], d))
    for l in range(1, d + 1):
        part = A[:, ell == l].sum(axis=1)
        out[:, l - 1] = np.where(var > 0, part / np.where(var > 0, var, 1.0), 0.0)
    return out
