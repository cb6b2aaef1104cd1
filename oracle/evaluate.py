"""Oracle: evaluation of the usFFT approximant (test infrastructure only).

eq. eval_formula with the identity periodization of the periodic model
(P:262-265):
    u^usFFT_{x_g}(y) = sum_{k in I} c_k(u_{x_g}) e^{2 pi i k . y}.
"""
from __future__ import annotations

import numpy as np


def evaluate(I: np.ndarray, C: np.ndarray, Y: np.ndarray) -> np.ndarray:
    """Complex [G][n]: direct double sum over k for every node g and point y_j (Y is [d][n])."""
    I = np.asarray(I, dtype=np.float64)            # [nI][d]
    C = np.asarray(C, dtype=np.complex128)         # [G][nI]
    Y = np.asarray(Y, dtype=np.float64)            # [d][n]
    phase = 2.0 * np.pi * (I @ Y)                  # [nI][n]
    E = np.exp(1j * phase)
    return C @ E
