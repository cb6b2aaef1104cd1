"""Pins of oracle/cover.py (Step 3 multiple-R1L cover; accuracy metric P:885-891)
against what the paper, SPEC and the mathematics fix — not against the oracle's own formulas."""
import math

import numpy as np
import pytest

from oracle import cover
from usfft_inputs.fixtures import trig_poly


def _random_set(seed, n, d, N):
    rng = np.random.default_rng(seed)
    out, seen = [], set()
    while len(out) < n:
        k = tuple(int(v) for v in rng.integers(-N, N + 1, size=d))
        if k not in seen:
            seen.add(k)
            out.append(k)
    return np.array(out, dtype=np.int64)


def _residue(k, z, M):
    return sum(int(a) * int(b) for a, b in zip(k, z)) % M


def test_singleton_cover():
    """singleton set -> one lattice, one assignment; M > N (Z26)."""
    lat, assign, binv = cover.build_cover(np.array([[3, -1]]), seed=7, N=4)
    assert len(lat) == 1 and assign.tolist() == [0]
    M, z = lat[0]
    assert M > 4 and binv[0] == _residue((3, -1), z, M)


def test_cover_lattice_count_near_remark4():
    """Remark 4: with lattices of size ~ 4 (|I| - 1) about ceil(2 ln(2|I|)) of them
    cover I; every lattice has M >= 4 (|I| - 1)."""
    I = _random_set(21, 200, 5, 32)
    lat, _, _ = cover.build_cover(I, seed=21, N=32)
    assert all(M >= 4 * 199 for M, _ in lat)
    assert len(lat) <= math.ceil(2 * math.log(2 * 200))


@pytest.mark.parametrize("n,d,N,seed", [(100, 5, 16, 1), (37, 3, 8, 2), (250, 6, 32, 3)])
def test_cover_alias_free_against_full_set(n, d, N, seed):
    """S:154 and invariant S:186: every frequency is assigned to a lattice on which its residue
    differs from the residue of EVERY other member of the set (brute force over pairs)."""
    I = _random_set(seed, n, d, N)
    lat, assign, binv = cover.build_cover(I, seed=seed, N=N)
    assert (assign >= 0).all()
    for a in range(n):
        M, z = lat[assign[a]]
        ra = _residue(I[a], z, M)
        assert binv[a] == ra
        for b in range(n):
            if b != a:
                assert _residue(I[b], z, M) != ra
    for M, z in lat:                                   # prime sizes, z in [1, M-1]^d
        assert all(M % p for p in range(2, int(math.isqrt(M)) + 1))
        assert all(1 <= v < M for v in z) and len(z) == d


def test_cover_size_within_remark4_bound():
    """Remark 4: total nodes M <= ceil(2 ln(2|I|)) * 4 (|I| - 1) (typical case)."""
    I = _random_set(11, 100, 5, 16)
    lat, _, _ = cover.build_cover(I, seed=11, N=16)
    assert sum(M for M, _ in lat) <= math.ceil(2 * math.log(2 * 100)) * 4 * 99


@pytest.mark.parametrize("real", [False, True])
def test_exact_recovery_on_supported_polynomials(real):
    """S:170 / Step 3: for G polynomials supported on I, the cover coefficients equal the
    polynomials' coefficients (lattice exponential orthogonality on alias-free residues)."""
    tp = trig_poly(5, d=4, N=8, G=3, n_terms=41, real=real)
    lat, assign, binv = cover.build_cover(tp.freqs, seed=5, N=8)
    C, n_samples = cover.cover_coefficients(tp, tp.freqs, lat, assign, binv)
    assert n_samples == sum(M for M, _ in lat)
    assert np.abs(C - tp.coefs).max() <= 1e-12


def test_zero_samples_give_zero_coefficients():
    """S:171."""
    I = _random_set(4, 20, 3, 6)
    lat, assign, binv = cover.build_cover(I, seed=4, N=6)
    C, _ = cover.cover_coefficients(lambda Y: np.zeros((2, Y.shape[1])), I, lat, assign, binv)
    assert not C.any()


def test_error_metric_closed_forms():
    """P:885-891 on closed forms: a constant offset c gives err_1 = err_2 = err_inf = |c|; one
    spike s among n points gives s/n, s/sqrt(n), s; complex differences use the modulus."""
    n = 400
    ref = np.linspace(-1, 1, n)[None, :].repeat(2, 0)
    e = cover.errors(ref, ref + 0.25)
    assert np.allclose(e, 0.25, rtol=0, atol=1e-15)
    spike = ref.copy()
    spike[:, 17] += 3.0
    e = cover.errors(ref, spike)
    assert np.allclose(e[0], [3.0 / n, 3.0 / math.sqrt(n), 3.0], rtol=1e-14, atol=0)
    e = cover.errors(np.zeros((1, 2)), np.array([[3 + 4j, -3 - 4j]]))
    assert np.allclose(e, 5.0)
