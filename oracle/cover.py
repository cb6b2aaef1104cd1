"""Oracle: Step 3 of Alg. 1 and the accuracy metric (test infrastructure only, see
oracle/__init__.py).

Step 3: "Generate a sampling set X ⊂ T^d for I^(1,...,d) such that the corresponding
Fourier matrix A(X, I) is of full column rank and its pseudoinverse can be applied efficiently",
then "compute the corresponding Fourier coefficients" for every chi_g.  The paper realises X by
the multiple rank-1 lattice approach of [KaPoVo17, Alg. 1] / [Kae17] (Remark 4
P:1662: "working with c = 2 and delta = 0.5").  Reading Z26, in the form of
SPEC build_cover / cover_coefficients:

  * every lattice has size M = the smallest prime >= max(4 (|I| - 1), N + 1) with M - 1
    7-smooth: Remark 4's c / delta = 2 / 0.5 lattices of size ~ 4 (|I| - 1), on Z2's
    FFT-friendly sizes.  (SPEC's M > 2|R| for the unassigned rest R cannot work with
    uniqueness against the full set once |R| << |I|: no residue of a small lattice is unique.);
  * while frequencies of I remain unassigned (the set R): draw z in [1, M-1]^d with the
    counter-based generator (Z4, tag 5: t = d, i = lattice index q, l = attempt) and assign
    every k in R whose residue k.z mod M is unique among the residues of the FULL set I on
    this lattice (first lattice wins); a draw that assigns nothing is redrawn, at
    most 100 times in a row.  With M >= 4 (|I| - 1) a frequency is alias-free on a
    lattice with probability ~ e^(-1/4), so about ceil(2 ln(2|I|)) lattices suffice;
  * the lattice nodes are y_i = (i z mod M) / M, i = 0..M-1, in all d components (X ⊂ T^d has
    no random part);
  * the coefficient of k is (1/M) sum_i u(y_i) e^{-2 pi i i b / M} with b = k.z mod M on its
    lattice, which is exact for u supported on I: on that lattice no other
    frequency of I shares b.

Accuracy metric: for every node chi_g, over n_test parameter draws y^(j),
    err_p(x_g) = ( (1/n_test) sum_j |u_check(x_g, y^(j)) - u^usFFT(x_g, y^(j))|^p )^(1/p),
    err_inf(x_g) = max_j |u_check - u^usFFT|,
with u_check the FE solution at y^(j) and u^usFFT the approximant sum_k c_k e^{2 pi i k.y}.
"""
from __future__ import annotations

import numpy as np

from . import dft, lattice, plan

TAG_COVER = 5
MAX_EMPTY_DRAWS = 100


def cover_size(nI: int, N: int) -> int:
    """M of every cover lattice (Z26): smallest prime >= max(4 (|I| - 1), N + 1), M-1 7-smooth."""
    return plan.next_lattice_prime(max(4 * (nI - 1), N + 1))


def cover_z(seed: int, d: int, q: int, attempt: int, M: int) -> list[int]:
    """Generating vector of cover lattice q (1-based), draw `attempt` (0-based) (Z4, Z26)."""
    return [1 + plan.draw(seed, TAG_COVER, d, q, attempt, j) % (M - 1) for j in range(1, d + 1)]


def build_cover(I, seed: int, N: int):
    """Multiple-R1L cover of I (Z26).  Returns (lattices [(M, z)], assign int [nI], bin int [nI]):
    frequency a is read on lattice assign[a] at bin[a]."""
    I = np.asarray(I, dtype=np.int64).reshape(len(I), -1)
    nI, d = I.shape
    assign = np.full(nI, -1, dtype=np.int64)
    binv = np.zeros(nI, dtype=np.int64)
    lattices = []
    empty = 0
    attempt = 0
    M = cover_size(nI, N)
    while (assign < 0).any():
        z = cover_z(seed, d, len(lattices) + 1, attempt, M)
        attempt += 1
        b = lattice.bins(I, [z], M)[0]                   # residues of the FULL set
        unique = np.bincount(b, minlength=M)[b] == 1
        new = unique & (assign < 0)
        if not new.any():
            empty += 1
            if empty > MAX_EMPTY_DRAWS:
                raise RuntimeError("cover construction: 100 consecutive empty draws")
            continue
        empty = 0
        attempt = 0
        assign[new] = len(lattices)
        binv[new] = b[new]
        lattices.append((M, z))
    return lattices, assign, binv


def cover_nodes(M: int, z, d: int) -> np.ndarray:
    """Nodes of one cover lattice, fp64 [d][M] (all d components from the lattice)."""
    return lattice.nodes(M, [z], np.zeros(d), d)


def cover_coefficients(blackbox, I, lattices, assign, binv):
    """c_{k,g} for every k in I and node g: complex [G][nI]; also the number of samples."""
    I = np.asarray(I, dtype=np.int64).reshape(len(I), -1)
    d = I.shape[1]
    C = None
    n_samples = 0
    for q, (M, z) in enumerate(lattices):
        U = blackbox(cover_nodes(M, z, d))               # [G][M]
        n_samples += M
        if C is None:
            C = np.zeros((U.shape[0], I.shape[0]), dtype=np.complex128)
        sel = np.nonzero(assign == q)[0]
        C[:, sel] = dft.lattice_dft(U, M, binv[sel])
    return C, n_samples


def errors(U_check: np.ndarray, U_approx: np.ndarray) -> np.ndarray:
    """[G][3] = (err_1, err_2, err_inf) per node; U_* are [G][n_test]."""
    D = np.abs(np.asarray(U_check) - np.asarray(U_approx))
    return np.stack([D.mean(axis=1), np.sqrt((D * D).mean(axis=1)), D.max(axis=1)], axis=1)
