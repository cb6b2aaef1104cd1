"""Seeded synthetic black boxes and points (no usFFT arithmetic).

A ``TrigPoly`` is G multivariate trigonometric polynomials p^(g)(y) = sum_k p_k^(g) e^{2 pi i k.y}
with supports in [-N, N]^d (Thm 1.1 setting).  ``real=True`` closes every support
under k -> -k with conjugate coefficients so the samples are real (the PDE samples are real).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class TrigPoly:
    freqs: np.ndarray        # int64 [n_terms][d]
    coefs: np.ndarray        # complex128 [G][n_terms]
    real: bool = False       # conjugate-closed support -> real samples

    def __call__(self, Y: np.ndarray) -> np.ndarray:
        """Samples [G][B] at the nodes Y [d][B] (complex, or real if conjugate-closed)."""
        Y = np.asarray(Y, dtype=np.float64)
        E = np.exp(2j * np.pi * (self.freqs.astype(np.float64) @ Y))
        out = self.coefs @ E
        if self.real:
            return np.ascontiguousarray(out.real)
        return out


def trig_poly(seed: int, d: int, N: int, G: int, n_terms: int, real: bool = True,
              min_abs: float = 0.5, max_active: int | None = None) -> TrigPoly:
    """G polynomials sharing a random support of n_terms distinct frequencies in [-N, N]^d.

    Each node gets its own random coefficients with |p_k| in [min_abs, 1].  With real=True the
    support is closed under negation (0 stays single and real) and n_terms counts all members.
    ``max_active`` limits the number of nonzero components per frequency (P:137 notes <= 4).
    """
    rng = np.random.default_rng(seed)
    freqs: list[tuple] = []
    seen = set()
    while len(freqs) < n_terms:
        if real and n_terms - len(freqs) == 1:          # odd count: fill with k = 0 if free
            z0 = (0,) * d
            if z0 not in seen:
                seen.add(z0)
                freqs.append(z0)
            break
        k = np.zeros(d, dtype=np.int64)
        na = d if max_active is None else int(rng.integers(1, max_active + 1))
        dims = rng.choice(d, size=min(na, d), replace=False)
        k[dims] = rng.integers(-N, N + 1, size=dims.shape[0])
        key = tuple(int(v) for v in k)
        if key in seen:
            continue
        if real:
            neg = tuple(-v for v in key)
            if key != neg and len(freqs) + 2 > n_terms:
                continue
            seen.add(key)
            seen.add(neg)
            freqs.append(key)
            if key != neg:
                freqs.append(neg)
        else:
            seen.add(key)
            freqs.append(key)
    F = np.asarray(freqs, dtype=np.int64)
    mag = rng.uniform(min_abs, 1.0, size=(G, F.shape[0]))
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(G, F.shape[0]))
    C = mag * np.exp(1j * ph)
    if real:
        index = {tuple(int(v) for v in F[q]): q for q in range(F.shape[0])}
        for q in range(F.shape[0]):
            key = tuple(int(v) for v in F[q])
            neg = tuple(-v for v in key)
            p = index[neg]
            if p == q:
                C[:, q] = mag[:, q]                           # zero frequency: real
            elif p > q:
                C[:, p] = np.conj(C[:, q])
    return TrigPoly(F, C, real)


def uniform_points(seed: int, d: int, n: int) -> np.ndarray:
    """n seeded points uniform on [0,1)^d, layout [d][n]."""
    rng = np.random.default_rng(seed)
    return rng.random((d, n))
