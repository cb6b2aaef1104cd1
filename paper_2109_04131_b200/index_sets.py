"""A-priori frequency sets for the comparison of Sec. 4.5: axis cross, hyperbolic
crosses (uniform weight 1/4 or weights 1/j^q) and weighted l1-balls.  Coefficients on such a set
come from Step 3 alone (`Detector.step3`), i.e. Alg. 1 with Steps 1-2 skipped.

Host enumeration with integer budgets (no floating point): the product constraint
prod_j f_j <= N is enumerated as f_1 <= N, prod_{j>1} f_j <= floor(N / f_1).  Rows come out in
lexicographic order; k = 0 is always included (reading Z31).
"""
from __future__ import annotations

import numpy as np

KINDS = ("axis", "hc_uniform", "hc", "l1")


def _mult(kind: str, j: int, q: int) -> int:
    """1 / weight of dimension j (1-based)."""
    return 4 if kind == "hc_uniform" else j ** q


def frequency_set(kind: str, d: int, N: int, q: int = 1, limit: int = 5_000_000) -> np.ndarray:
    """int64 [n][d], lexicographically sorted; raises if more than `limit` rows."""
    if kind not in KINDS:
        raise ValueError(f"unknown set kind {kind!r}")
    rows: list[tuple[int, ...]] = []
    if kind == "axis":
        for j in range(d):
            for v in range(-N, N + 1):
                k = [0] * d
                k[j] = v
                rows.append(tuple(k))
        rows = sorted(set(rows))
        return np.array(rows, dtype=np.int64).reshape(-1, d)
    prod = kind in ("hc_uniform", "hc")
    cur = [0] * d

    def rec(j: int, budget: int):
        if len(rows) > limit:
            raise ValueError(f"frequency set larger than {limit}")
        if j == d:
            rows.append(tuple(cur))
            return
        m = _mult(kind, j + 1, q)
        vmax = budget // m                      # |k_j| with m |k_j| <= budget
        for v in range(-vmax, vmax + 1):
            cur[j] = v
            if v == 0:
                rec(j + 1, budget)
            else:
                rec(j + 1, budget // (m * abs(v)) if prod else budget - m * abs(v))
        cur[j] = 0

    rec(0, N)
    return np.array(rows, dtype=np.int64).reshape(-1, d)
