"""Pins for oracle/plan.py and oracle/lattice.py (CPU only)."""
import json
import math
import os

import numpy as np
import pytest

from oracle import lattice, plan

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_splitmix64_published_output():
    g = GOLD["splitmix64"][0]
    assert plan.sm64(g["state"]) == int(g["output"], 16)


def test_u01_range_and_uniformity():
    xs = np.array([plan.u01(plan.draw(3, 1, t, i, 0, j)) for t in range(1, 11)
                   for i in range(1, 11) for j in range(1, 41)])
    assert xs.min() >= 0.0 and xs.max() < 1.0
    assert abs(xs.mean() - 0.5) < 0.03                      # 4000 draws: sd of mean ~ 0.0046
    hist = np.histogram(xs, bins=10, range=(0, 1))[0]
    assert hist.min() > 300 and hist.max() < 500


def test_draws_are_counter_based():
    # changing one counter changes the draw; re-evaluation is deterministic
    a = plan.draw(1, 3, 2, 1, 0, 1)
    assert a == plan.draw(1, 3, 2, 1, 0, 1)
    assert len({a, plan.draw(1, 3, 2, 1, 0, 2), plan.draw(1, 3, 2, 1, 1, 1),
                plan.draw(1, 3, 2, 2, 0, 1), plan.draw(1, 3, 3, 1, 0, 1),
                plan.draw(1, 2, 2, 1, 0, 1), plan.draw(2, 3, 2, 1, 0, 1)}) == 7


def _brute_prime(n):
    return n >= 2 and all(n % f for f in range(2, int(math.isqrt(n)) + 1))


def _brute_smooth(n):
    return all(p in (2, 3, 5, 7) for p in range(2, n + 1) if n % p == 0 and _brute_prime(p))


@pytest.mark.parametrize("lo", [3, 50, 80, 400, 1000, 2000, 4000])
def test_next_lattice_prime_brute_force(lo):
    p = plan.next_lattice_prime(lo)
    assert _brute_prime(p) and _brute_smooth(p - 1)
    for q in range(lo, p):
        assert not (_brute_prime(q) and _brute_smooth(q - 1))


def test_lattice_sizes_of_configs():
    # Z2 rule evaluated by hand: 97-1 = 2^5*3, 401-1 = 2^4*5^2, 2017-1 = 2^5*3^2*7, 4001-1 = 2^5*5^3
    assert plan.lattice_size(20, 8) == 97
    assert plan.lattice_size(100, 32) == 401
    assert plan.lattice_size(500, 64) == 2017
    assert plan.lattice_size(1000, 64) == 4001


@pytest.mark.parametrize("nJ", [1, 2, 17, 105, 1500, 10 ** 6])
def test_num_lattices(nJ):
    L = plan.num_lattices(nJ)
    assert L % 2 == 1 and L >= 2 * math.log(2 * nJ) and L <= 2 * math.log(2 * nJ) + 2


def test_z_range():
    z = plan.z_vectors(5, 4, 2, 401, 17)
    assert len(z) == 17 and all(len(r) == 4 for r in z)
    assert min(min(r) for r in z) >= 1 and max(max(r) for r in z) <= 400


@pytest.mark.parametrize("ex", GOLD["lattice_nodes"])
def test_spec_lattice_nodes(ex):
    y = lattice.nodes(ex["M"], [ex["z"]], [0.0, 0.0], 2)
    assert np.allclose(y[:, ex["i"]], ex["node"], atol=1e-15)


@pytest.mark.parametrize("ex", GOLD["residues"])
def test_spec_residues(ex):
    assert lattice.bins(np.array(ex["set"]), [ex["z"]], ex["M"])[0].tolist() == ex["bins"]


@pytest.mark.parametrize("ex", GOLD["injective"])
def test_spec_injective(ex):
    b = lattice.bins(np.array(ex["set"]), [ex["z"]], ex["M"])[0]
    assert lattice.injective(b) == ex["injective"]


def test_nodes_and_bins_satisfy_exact_phase_identity():
    """k . y_i = i * b(k) / M (mod 1) as an exact integer identity: y_i*M is the integer
    (i z mod M) and sum_j k_j (i z_j mod M) = i (k.z) (mod M)."""
    rng = np.random.default_rng(0)
    for M in (5, 97, 401):
        t = 4
        z = rng.integers(1, M, size=(3, t)).tolist()
        J = rng.integers(-8, 9, size=(20, t))
        y = lattice.nodes(M, z, [0.5] * 6, t)
        b = lattice.bins(J, z, M)
        for l in range(3):
            for i in (0, 1, 2, M // 2, M - 1):
                n = y[:t, l * M + i] * M
                nint = np.rint(n).astype(np.int64)
                assert np.all(np.abs(n - nint) < 1e-9)
                assert nint.tolist() == [(i * zz) % M for zz in z[l]]
                lhs = (J @ nint) % M
                rhs = (i * b[l]) % M
                assert np.array_equal(lhs, rhs)
            assert np.all(y[t:, l * M:(l + 1) * M] == 0.5)


def test_coordinate_bijection_prime_M():
    """for prime M and z_j != 0 mod M, {y_{i,j}} = {n/M}."""
    M = 97
    y = lattice.nodes(M, [[5, 31, 96]], [0.0] * 3, 3)
    for j in range(3):
        assert sorted(np.rint(y[j] * M).astype(int).tolist()) == list(range(M))


def test_step1_line_nodes():
    K = 17
    xs = [0.1, 0.2, 0.3, 0.4]
    y = lattice.nodes(K, [[1]], xs, 1, line_axis=2)
    assert np.allclose(y[2], np.arange(K) / K)
    for j in (0, 1, 3):
        assert np.all(y[j] == xs[j])


def test_candidate_order():
    J = lattice.candidates(np.array([[1, 2], [3, 4]]), np.array([-1, 0, 5]))
    assert J.tolist() == [[1, 2, -1], [1, 2, 0], [1, 2, 5], [3, 4, -1], [3, 4, 0], [3, 4, 5]]
