"""Oracle: the a-priori frequency sets of the paper's comparison (Sec. 4.5 "Comparison to given
frequency sets"), by brute force over the box [-N, N]^d (test infrastructure only,
see oracle/__init__.py).  Every set contains k = 0 (reading Z31).

    axis      {k : ||k||_0 <= 1, ||k||_1 <= N}
    hc_uniform{k : prod_j max(1, 4 |k_j|) <= N}            (uniform weight 1/4)
    hc_q      {k : prod_j max(1, j^q |k_j|) <= N}          (weights 1/j^q, q = 1, 2)
    l1_q      {k : sum_j j^q |k_j| <= N}                   (weights 1/j^q, q = 1, 2)
"""
from __future__ import annotations

import itertools

import numpy as np


def member(kind: str, k, N: int, q: int = 1) -> bool:
    k = [abs(int(v)) for v in k]
    if kind == "axis":
        return sum(v != 0 for v in k) <= 1 and sum(k) <= N
    if kind == "hc_uniform":
        return float(np.prod([max(1, 4 * v) for v in k])) <= N
    if kind == "hc":
        return float(np.prod([max(1, (j + 1) ** q * v) for j, v in enumerate(k)])) <= N
    if kind == "l1":
        return sum((j + 1) ** q * v for j, v in enumerate(k)) <= N
    raise ValueError(kind)


def brute_force(kind: str, d: int, N: int, q: int = 1) -> np.ndarray:
    """All members in lexicographic order of the box [-N, N]^d (small d and N only)."""
    out = [k for k in itertools.product(range(-N, N + 1), repeat=d) if member(kind, k, N, q)]
    return np.array(out, dtype=np.int64).reshape(-1, d)
