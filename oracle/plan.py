"""Oracle: the random round plan of Alg. 1 (test infrastructure only, see oracle/__init__.py).

Alg. 1 draws, per detection round (t, i):
  * Step 1 & 2a (Alg. 1): x'_j in T uniformly at random for j != t, and the line
    nodes x^(l) with l/K_t in slot t, K_t = 2N+1;
  * Step 2 (Alg. 1): x'_{t+1..d} uniformly at random, and a sampling set X for J_t
    "that allows for the application of Algorithm A".  With Algorithm A = random
    rank-1 lattices this is L rank-1 lattices Lambda(z_l, M) (R1L).

The paper fixes neither the generator nor the lattice sizes; DESIGN.md §3 readings:
  Z4  counter-based SplitMix64 draws, h = sm64(sm64(sm64(sm64(sm64(seed)^tag)^t)^i)^((l<<20)^j))
      with 1-based t, i, j and 0-based l; x' = (h>>11)*2^-53; z = 1 + h mod (M-1) (Z3).
      Tags: 1 Step-1 shift, 2 Step-2 shift, 3 lattice vectors z, 4|(M<<8) mode-R tries.
  Z2  M = smallest prime p >= max(4*s_tilde, K+1) with p-1 7-smooth (M prime: Lemma P:847,
      P:878); L = ceil(2 ln(2|J_t|)), made odd (mirrors ceil(2 ln(2|I|)) of Remark 4).
      Mode R (single reconstructing R1L, Table 1 row 1 P:242): primes with
      p-1 7-smooth ascending from max(2|J|, N+1), <= 50 tries of z per prime, M <= 2^26.
"""
from __future__ import annotations

import math

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

TAG_STEP1_SHIFT = 1
TAG_STEP2_SHIFT = 2
TAG_Z = 3
TAG_MODE_R = 4

MODE_R_TRIES = 50
MODE_R_MAX_M = 1 << 26


def sm64(x: int) -> int:
    """SplitMix64 output for state x (Steele/Lea/Flood 2014; Vigna's splitmix64.c)."""
    z = (x + GOLDEN) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def draw(seed: int, tag: int, t: int, i: int, l: int, j: int) -> int:
    """Counter-based 64-bit draw (reading Z4): no sequential state."""
    h = sm64(seed & MASK64)
    h = sm64(h ^ (tag & MASK64))
    h = sm64(h ^ (t & MASK64))
    h = sm64(h ^ (i & MASK64))
    return sm64(h ^ (((l << 20) ^ j) & MASK64))


def u01(h: int) -> float:
    """Uniform double in [0, 1) from the top 53 bits (Z4)."""
    return float(h >> 11) * 2.0 ** -53


def is_prime(n: int) -> bool:
    """Trial division (n < 2^27 here)."""
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    f = 3
    while f * f <= n:
        if n % f == 0:
            return False
        f += 2
    return True


def is_7smooth(n: int) -> bool:
    for p in (2, 3, 5, 7):
        while n % p == 0 and n > 1:
            n //= p
    return n == 1


def next_lattice_prime(lo: int) -> int:
    """Smallest prime p >= lo with p-1 7-smooth (Z2)."""
    p = max(lo, 3)
    while not (is_prime(p) and is_7smooth(p - 1)):
        p += 1
    return p


def lattice_size(s_tilde: int, N: int) -> int:
    """M of a Step-2 round (Z2): smallest such prime >= max(4 s_tilde, K+1), K = 2N+1."""
    return next_lattice_prime(max(4 * s_tilde, 2 * N + 2))


def num_lattices(nJ: int) -> int:
    """L of a Step-2 round (Z2): ceil(2 ln(2|J|)), made odd; at least 1."""
    L = max(1, math.ceil(2.0 * math.log(2.0 * nJ)))
    if L % 2 == 0:
        L += 1
    return L


def shift(seed: int, step: int, t: int, i: int, d: int) -> list[float]:
    """The random components x'_j, j = 1..d, of round (t, i) (P:287 / P:307).

    All d components are drawn; Step 1 uses j != t, Step 2 uses j > t (one x' per round,
    shared by every lattice and every node chi_g: Z8).
    """
    tag = TAG_STEP1_SHIFT if step == 1 else TAG_STEP2_SHIFT
    return [u01(draw(seed, tag, t, i, 0, j)) for j in range(1, d + 1)]


def z_vectors(seed: int, t: int, i: int, M: int, L: int) -> list[list[int]]:
    """Generating vectors z_l in [1, M-1]^t of the L random R1Ls of round (t, i) (Z3, Z4)."""
    return [[1 + draw(seed, TAG_Z, t, i, l, j) % (M - 1) for j in range(1, t + 1)]
            for l in range(L)]


def mode_r_z(seed: int, t: int, i: int, M: int, trial: int) -> list[int]:
    """Mode-R candidate z of try `trial` at lattice size M (Z2)."""
    tag = TAG_MODE_R | (M << 8)
    return [1 + draw(seed, tag, t, i, trial, j) % (M - 1) for j in range(1, t + 1)]
