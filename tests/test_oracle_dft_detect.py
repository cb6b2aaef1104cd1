"""Pins for oracle/dft.py, oracle/detect.py, oracle/usfft.py, oracle/evaluate.py (CPU only)."""
import itertools
import json
import os

import numpy as np
import pytest

from oracle import detect, dft, evaluate, lattice, plan, usfft
from usfft_inputs import trig_poly

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------------------ lattice DFT
def test_orthogonality():
    """(1/M) sum_i e^{2 pi i i h / M} e^{-2 pi i i b / M} = [h = b mod M]."""
    M = 13
    i = np.arange(M)
    U = np.exp(2j * np.pi * np.outer(np.arange(M), i) / M)        # rows: pure tones h
    V = dft.lattice_dft(U, M, np.arange(M))
    assert np.abs(V - np.eye(M)).max() < 1e-14


@pytest.mark.parametrize("ex", GOLD["lattice_coefficients"])
def test_spec_lattice_coefficients(ex):
    M, z = ex["M"], [ex["z"]]
    y = lattice.nodes(M, z, [0.0, 0.0], 2)
    F = np.array([t[0] for t in ex["terms"]])
    C = np.array([[complex(*t[1]) for t in ex["terms"]]])
    u = C @ np.exp(2j * np.pi * (F @ y))
    b = lattice.bins(np.array(ex["set"]), z, M)[0]
    got = dft.lattice_dft(u, M, b)[0]
    want = np.array([complex(*c) for c in ex["coef"]])
    assert np.abs(got - want).max() < 1e-14


def test_exact_recovery_on_reconstructing_lattice():
    """lattice DFT of a trig polynomial supported on a set J for which the
    lattice is reconstructing returns its coefficients exactly (100 random fixtures)."""
    rng = np.random.default_rng(11)
    for rep in range(100):
        d, N = 3, 6
        tp = trig_poly(1000 + rep, d, N, 2, 12, real=False)
        J = tp.freqs
        for trial in range(200):                       # search a reconstructing z
            M = plan.next_lattice_prime(int(rng.integers(60, 400)))
            z = rng.integers(1, M, size=d).tolist()
            b = lattice.bins(J, [z], M)[0]
            if lattice.injective(b):
                break
        else:
            pytest.fail("no reconstructing lattice found")
        y = lattice.nodes(M, [z], [0.0] * d, d)
        got = dft.lattice_dft(tp(y), M, b)
        assert np.abs(got - tp.coefs).max() < 1e-12


@pytest.mark.parametrize("t", [1, 2, 3])
def test_brute_force_tensor_grid(t):
    """Tier pin: for a trig polynomial with support in [-N,N]^t, (i) the full K^t tensor-grid
    DFT (np.fft.fftn), (ii) the lattice z = (1, K, K^2, ..), M = K^t and (iii) a mode-R random
    reconstructing lattice all give the same coefficients."""
    N = 3
    K = 2 * N + 1
    tp = trig_poly(7 + t, t, N, 3, 9 if t > 1 else 5, real=True)
    J = np.array(list(itertools.product(range(-N, N + 1), repeat=t)))
    # (i) tensor grid
    grid = np.meshgrid(*[np.arange(K) / K] * t, indexing="ij")
    Yg = np.stack([g.reshape(-1) for g in grid])
    Ug = tp(Yg).reshape((3,) + (K,) * t)
    Fg = np.fft.fftn(Ug, axes=tuple(range(1, t + 1))) / K ** t
    ref = np.stack([Fg[(slice(None),) + tuple(int(v) % K for v in k)] for k in J], axis=1)
    # (ii) Korobov-type lattice: k.z = sum k_j K^j is injective on [-N,N]^t mod K^t
    M = K ** t
    z = [[K ** j for j in range(t)]]
    y = lattice.nodes(M, z, [0.0] * t, t)
    b = lattice.bins(J, z, M)[0]
    assert lattice.injective(b)
    got = dft.lattice_dft(tp(y), M, b)
    assert np.abs(got - ref).max() < 1e-12
    # (iii) mode-R random lattice
    Mr, zr = usfft.mode_r_lattice(J, 5, t, 1, N)
    yr = lattice.nodes(Mr, zr, [0.0] * t, t)
    br = lattice.bins(J, zr, Mr)[0]
    got_r = dft.lattice_dft(tp(yr), Mr, br)
    assert np.abs(got_r - ref).max() < 1e-12
    # and the polynomial's own coefficients
    pos = {tuple(k): q for q, k in enumerate(J.tolist())}
    cols = [pos[tuple(k)] for k in tp.freqs.tolist()]
    assert np.abs(ref[:, cols] - tp.coefs).max() < 1e-12


# ------------------------------------------------------------------------------ detection
def test_select_brute_force():
    """Per-g top-s~ by (kappa desc, index asc), >= theta^2, > 0: brute force by enumerating
    rank positions (itertools over the tie-broken total order)."""
    rng = np.random.default_rng(2)
    for rep in range(50):
        G, nJ, s = 3, 9, int(rng.integers(1, 6))
        km = rng.choice([0.0, 0.5, 1.0, 2.0, 3.0, 1e-14], size=(G, nJ))
        th2 = float(rng.choice([0.0, 0.6, 1e-13]))
        D, votes = detect.select(km, s, th2)
        for g in range(G):
            # rank of j = number of candidates strictly before it in the total order
            rank = [sum(1 for q in range(nJ) if (km[g, q] > km[g, j]) or (km[g, q] == km[g, j] and q < j))
                    for j in range(nJ)]
            want = [j for j in range(nJ) if rank[j] < s and km[g, j] >= th2 and km[g, j] > 0]
            assert D[g].tolist() == want
        assert votes.tolist() == [sum(j in D[g] for g in range(G)) for j in range(nJ)]


def test_theta_relative():
    km = np.array([[4.0, 1e-12, 3.9e-12], [0.0, 2.0, 1.0]])
    th2 = detect.theta_squared(km, 1e-6)
    assert th2 == (1e-6 * 1e-6) * 4.0
    D, _ = detect.select(km, 3, th2)
    assert D[0].tolist() == [0] and D[1].tolist() == [1, 2]
    assert detect.theta_squared(km, 1e-6, theta_abs=0.5) == 0.25


def test_kappa_min_and_resolve_alias_free():
    """A 2-sparse signal seen through 3 lattices where lattice 0 aliases the pair: kappa_min is
    the clean value of lattice 1; resolve picks l* = 1 (first alias-free) for both."""
    # candidate bins per lattice (L=3, |J|=4); D_g = {0, 1}
    bins = np.array([[5, 5, 1, 2], [3, 4, 1, 2], [0, 1, 2, 3]])
    c = np.array([1.0 + 1.0j, 0.5 + 0.5j, 0, 0])          # constructive alias in lattice 0
    V = np.zeros((3, 1, 4), complex)
    for l in range(3):
        for k in range(4):
            V[l, 0, k] = sum(c[q] for q in range(2) if bins[l, q] == bins[l, k])
    km = detect.kappa_min(V)
    assert np.allclose(km[0], np.abs(c) ** 2)
    D = [np.array([0, 1])]
    coef, ls = detect.resolve(V, bins, D, np.array([0, 1, 2]))
    assert ls[0].tolist() == [1, 1, 0]
    assert np.allclose(coef[0], [1 + 1j, 0.5 + 0.5j, 0])


def test_resolve_median_fallback():
    bins = np.array([[0, 0], [1, 1], [2, 2]])        # both members collide in every lattice
    V = np.array([[[1.0 + 5j, 0]], [[3.0 + 1j, 0]], [[2.0 + 2j, 0]]])
    coef, ls = detect.resolve(V, bins, [np.array([0, 1])], np.array([0]))
    assert ls[0, 0] == -1 and coef[0, 0] == 2.0 + 2j


# ------------------------------------------------------------------------------ whole Alg. 1
@pytest.mark.parametrize("mode", ["A", "R"])
def test_spec_acceptance_exact_recovery(mode):
    """Thm 1.1 / SPEC acceptance 1: d = 6, Gamma = [-32,32]^6, G = 5,
    <= 20 terms, s = 20, r = 5: >= 18 of 20 trials recover all supports exactly and the
    coefficients to 1e-8."""
    ok = 0
    for trial in range(20):
        tp = trig_poly(500 + trial, 6, 32, 5, 20, real=False, max_active=4)
        cfg = dict(d=6, N=32, s=20, s_local=20, r=5, seed=trial, theta_rel=1e-6, mode=mode)
        res = usfft.run(cfg, tp)
        got = {tuple(k) for k in res["I"].tolist()}
        if got != {tuple(k) for k in tp.freqs.tolist()}:
            continue
        pos = {tuple(k): q for q, k in enumerate(res["I"].tolist())}
        cols = [pos[tuple(k)] for k in tp.freqs.tolist()]
        if np.abs(res["C"][:, cols] - tp.coefs).max() < 1e-8:
            ok += 1
    assert ok >= 18


def test_union_of_differing_supports():
    """G polynomials with pairwise different supports (Thm 1.1 allows disjoint I_g): the
    output is the union of all supports."""
    from usfft_inputs.fixtures import TrigPoly
    a = trig_poly(41, 4, 8, 1, 6, real=False)
    b = trig_poly(42, 4, 8, 1, 6, real=False)
    F = np.concatenate([a.freqs, b.freqs])
    C = np.zeros((2, F.shape[0]), complex)
    C[0, :6] = a.coefs[0]
    C[1, 6:] = b.coefs[0]
    tp = TrigPoly(F, C, False)
    res = usfft.run(dict(d=4, N=8, s=6, s_local=6, r=5, seed=3, theta_rel=1e-6, mode="A"), tp)
    assert {tuple(k) for k in res["I"].tolist()} == {tuple(k) for k in F.tolist()}


def test_zero_black_box():
    res = usfft.run(dict(d=3, N=4, s=5, s_local=5, r=2, seed=1, theta_rel=1e-6),
                    lambda Y: np.zeros((2, Y.shape[1])))
    # nothing passes (exact zeros are never detected), I^(t) = {0} per Z9, final set empty
    assert res["I"].shape[0] == 0


@pytest.mark.parametrize("ex", GOLD["detect_1d"])
def test_spec_detect_1d(ex):
    F = np.array([[t[0][0], 0] for t in ex["terms"]])
    C = np.array([[complex(*t[1]) for t in ex["terms"]]])
    from usfft_inputs.fixtures import TrigPoly
    tp = TrigPoly(F, C, False)
    log = []
    usfft.run(dict(d=2, N=ex["N"], s=3, s_local=3, r=1, seed=0, theta_rel=1e-6), tp, log)
    res = usfft.run(dict(d=2, N=ex["N"], s=3, s_local=3, r=1, seed=0, theta_rel=1e-6), tp)
    assert res["I1d"][0].tolist() == ex["detected"]
    assert abs(abs(res["C"][0, 0]) - ex["abs"]) < 1e-12


@pytest.mark.parametrize("ex", GOLD["evaluate"])
def test_spec_evaluate(ex):
    U = evaluate.evaluate(np.array(ex["I"]), np.array([[complex(*c) for c in ex["C"]]]),
                          np.array(ex["y"]).reshape(-1, 1))
    assert abs(U[0, 0] - complex(*ex["value"])) < 1e-15


# ---- Z25 fragile-decision rule (two-sided), pinned on hand-built key vectors ------------------
# Keys are given as magnitudes m (kappa = m^2); max m = 1 so eps = 1e-10 throughout.
def _frag(mags, s, theta=0.0):
    m = np.asarray(mags, dtype=np.float64)[None, :]
    return detect.fragile(m * m, s, theta * theta)[0].tolist()


def test_fragile_separated_keys_none():
    """Well separated keys and threshold: no decision is fragile, the cut element included (the
    one-sided rule of round 1 flagged the s~-th key itself)."""
    assert _frag([1.0, 0.5, 0.25, 0.125, 0.0625], 2, theta=0.01) == [False] * 5


def test_fragile_cross_cut_pair():
    """The 2nd (in) and 3rd (out) keys differ by 3e-11 < eps: exactly that pair is fragile."""
    assert _frag([1.0, 0.5, 0.5 - 3e-11, 0.125], 2) == [False, True, True, False]


def test_fragile_same_side_pair_not():
    """A near tie inside the selection (both in) or outside it (both out) cannot change D_g."""
    assert _frag([1.0, 1.0 - 3e-11, 0.5, 0.25, 0.25 - 3e-11], 2) == [False] * 5


def test_fragile_bit_equal_across_cut_not():
    """Bit-equal keys straddling the cut are ordered by index on both sides: not fragile; a
    different key within eps of them across the cut is."""
    assert _frag([1.0, 0.5, 0.5, 0.125], 2) == [False] * 4
    assert _frag([1.0, 0.5, 0.5, 0.5 - 2e-11], 3) == [False, True, True, True]


def test_fragile_threshold_band():
    """An 'in' key within eps of theta is fragile (the threshold decision, Z5); an 'out' key
    near theta is not (its rank already excludes it)."""
    assert _frag([1.0, 0.3 + 5e-11, 0.2, 0.1], 2, theta=0.3) == [False, True, False, False]
    assert _frag([1.0, 0.5, 0.3 + 5e-11, 0.1], 2, theta=0.3) == [False] * 4


def test_fragile_band_edge():
    """Differences just outside eps are not fragile; s~ >= |J| leaves no cut."""
    assert _frag([1.0, 0.5, 0.5 - 2e-10], 2) == [False] * 3
    assert _frag([1.0, 0.5 + 1e-12, 0.5], 5) == [False] * 3


def test_fragile_swaps_below_threshold_not():
    """A near tie across the cut between two keys below theta changes no D_g (neither is
    detected either way); the same tie above theta is fragile."""
    assert _frag([1.0, 0.5, 1e-3, 1e-3 - 2e-11], 3, theta=0.1) == [False] * 4
    assert _frag([1.0, 0.5, 0.2, 0.2 - 2e-11], 3, theta=0.1) == [False, False, True, True]


def test_fragile_keys_one_ulp_apart_with_equal_sqrt():
    """Equality is judged on the key kappa, not on m = sqrt(kappa): two keys one ulp apart whose
    square roots round to the same double straddle the cut -> fragile (the conjugate pair
    k, -k of a real sample set has such keys)."""
    k1 = 5.147219e-15
    k2 = np.nextafter(k1, 1.0)
    while np.sqrt(k2) != np.sqrt(k1):                  # find a pair with one shared sqrt
        k1 = np.nextafter(k1, 1.0)
        k2 = np.nextafter(k1, 1.0)
    K = np.array([[1.0, k1, k2, 1e-20]])
    fr = detect.fragile(K, 2, 0.0)[0].tolist()
    assert fr == [False, True, True, False]
