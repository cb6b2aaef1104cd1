"""Pins for oracle/fe.py: P1 FE black box (CPU only)."""
import json
import os

import numpy as np
import pytest
import scipy.special

from oracle import fe
from usfft_inputs import config

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _model(n, a_func, f_func):
    return dict(n=n, d=0, amp=[], theta="sin", form="affine", f=f_func, a_func=a_func)


def test_constant_coefficient_is_five_point_laplacian():
    """a = 1 on the "/" triangulation: P1 stiffness = textbook 5-point Laplacian (no h scaling in
    2-D), hypotenuse couplings vanish; centroid load of f = x2 is h^2 x2 at each node."""
    n = 6
    G = (n - 1) ** 2
    cx, cy = fe.centroids(n)
    ab, b = fe.assemble(n, np.ones_like(cx), cy.copy())
    A = fe.banded_to_dense(ab)
    ref = np.zeros((G, G))
    for j in range(1, n):
        for i in range(1, n):
            p = (j - 1) * (n - 1) + (i - 1)
            ref[p, p] = 4.0
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                ii, jj = i + di, j + dj
                if 1 <= ii <= n - 1 and 1 <= jj <= n - 1:
                    ref[p, (jj - 1) * (n - 1) + (ii - 1)] = -1.0
    assert np.abs(A - ref).max() < 1e-13
    x1, x2 = fe.node_coords(n)
    assert np.allclose(b, x2 / n ** 2, rtol=1e-13, atol=0)


def _order(errs, ns):
    return [np.log(errs[k] / errs[k + 1]) / np.log(ns[k + 1] / ns[k]) for k in range(len(ns) - 1)]


def test_manufactured_constant_coefficient_order2():
    """a = 1, f = 2 pi^2 sin(pi x1) sin(pi x2) -> u = sin sin; order >= 1.9."""
    ns = [8, 16, 32]
    errs = []
    for n in ns:
        m = _model(n, lambda x1, x2: np.ones_like(x1),
                   lambda x1, x2: 2 * np.pi ** 2 * np.sin(np.pi * x1) * np.sin(np.pi * x2))
        u = fe.solve(m, np.zeros(0))
        x1, x2 = fe.node_coords(n)
        errs.append(np.abs(u - np.sin(np.pi * x1) * np.sin(np.pi * x2)).max())
    assert min(_order(errs, ns)) >= 1.9


def test_manufactured_variable_coefficient_order2():
    """a = 1 + x1 x2 / 2, u = sin sin, f = -div(a grad u) in closed form."""
    def a(x1, x2):
        return 1.0 + 0.5 * x1 * x2

    def f(x1, x2):
        s1, s2 = np.sin(np.pi * x1), np.sin(np.pi * x2)
        c1, c2 = np.cos(np.pi * x1), np.cos(np.pi * x2)
        return a(x1, x2) * 2 * np.pi ** 2 * s1 * s2 - (0.5 * x2 * np.pi * c1 * s2 + 0.5 * x1 * np.pi * s1 * c2)

    ns = [8, 16, 32]
    errs = []
    for n in ns:
        u = fe.solve(_model(n, a, f), np.zeros(0))
        x1, x2 = fe.node_coords(n)
        errs.append(np.abs(u - np.sin(np.pi * x1) * np.sin(np.pi * x2)).max())
    assert min(_order(errs, ns)) >= 1.9


@pytest.mark.parametrize("cfg", [1, 2, 4])
def test_spd_m_matrix_and_residual(cfg):
    """Cholesky succeeds (SPD); f = x2 >= 0 gives u >= 0 (M-matrix); residual at round-off."""
    m = config(cfg)
    rng = np.random.default_rng(cfg)
    for _ in range(3):
        u, rr = fe.solve(m, rng.random(m["d"]), return_residual=True)
        assert np.all(u >= 0.0) and rr < 1e-11


def test_coefficient_maps():
    m = config(1)
    x1, x2 = np.random.default_rng(0).random((2, 50))
    assert np.allclose(fe.coefficient(m, np.zeros(4), x1, x2), 1.0, atol=0)
    ml = config(4)
    y = np.full(20, 0.5)                                                        # Phi^-1(1/2) = 0
    assert np.allclose(fe.coefficient(ml, y, x1, x2), 1.0, atol=0)
    assert fe.theta_map("probit", np.array([0.0]))[0] == -6.0                   # clip (Z15)
    assert abs(fe.theta_map("probit", np.array([0.975]))[0] - 1.959963984540054) < 1e-12
    # tent: phi(0) = alpha = -1, phi(1/2) = beta = 1 (A2); symmetric (A3)
    assert fe.theta_map("tent", np.array([0.0, 0.5, 0.25]))[0:3].tolist() == [-1.0, 1.0, 0.0]
    t = np.linspace(0, 0.5, 11)
    assert np.allclose(fe.theta_map("tent", 0.5 - t), fe.theta_map("tent", 0.5 + t))


@pytest.mark.parametrize("ex", GOLD["ellipticity"])
def test_paper_ellipticity_bounds(ex):
    """Periodic model of Sec. 4.2: a_min/max = 1 -/+ (c/sqrt6) zeta(mu); the
    oracle's coefficient stays inside the d-term bounds for random (x, y)."""
    z = scipy.special.zeta(ex["mu"])
    assert abs(1 - ex["c"] / np.sqrt(6) * z - ex["a_min"]) <= ex["tol"]
    assert abs(1 + ex["c"] / np.sqrt(6) * z - ex["a_max"]) <= ex["tol"]
    d = 10
    amp = [ex["c"] / np.sqrt(6) * j ** -ex["mu"] for j in range(1, d + 1)]
    m = dict(n=8, d=d, amp=amp, theta="sin", form="affine", f="x2")
    rng = np.random.default_rng(1)
    for _ in range(50):
        a = fe.coefficient(m, rng.random(d), *rng.random((2, 200)))
        assert a.min() >= 1 - sum(amp) - 1e-15 and a.max() <= 1 + sum(amp) + 1e-15


def test_stencil_derivation_matches_element_assembly():
    """Z11: the element-assembled matrix for arbitrary centroid values equals the 5-point stencil
    w_h(i,j) = (a(T_lo(i,j)) + a(T_up(i,j-1)))/2, w_v(i,j) = (a(T_up(i,j)) + a(T_lo(i-1,j)))/2.
    This checks the derivation the GPU path uses against textbook assembly."""
    n = 7
    G = (n - 1) ** 2
    rng = np.random.default_rng(3)
    a_T = rng.uniform(0.5, 2.0, size=2 * n * n)
    A = fe.banded_to_dense(fe.assemble(n, a_T, np.zeros_like(a_T))[0])

    def lo(ci, cj):
        return a_T[2 * (cj * n + ci)]

    def up(ci, cj):
        return a_T[2 * (cj * n + ci) + 1]

    def idx(i, j):
        return (j - 1) * (n - 1) + (i - 1) if 1 <= i <= n - 1 and 1 <= j <= n - 1 else -1

    R = np.zeros((G, G))
    for j in range(1, n):
        for i in range(1, n):
            p = idx(i, j)
            wE = (lo(i, j) + up(i, j - 1)) / 2
            wW = (lo(i - 1, j) + up(i - 1, j - 1)) / 2
            wN = (up(i, j) + lo(i - 1, j)) / 2
            wS = (up(i, j - 1) + lo(i - 1, j - 1)) / 2
            R[p, p] = wE + wW + wN + wS
            for q, w in ((idx(i + 1, j), wE), (idx(i - 1, j), wW), (idx(i, j + 1), wN), (idx(i, j - 1), wS)):
                if q >= 0:
                    R[p, q] = -w
    assert np.abs(A - R).max() < 1e-13


# ------------------------------------------------------------------ lognormal periodization (Z27)
def test_phi_delta_spec_examples_and_poles():
    """SPEC S:353-356 / P:500-515: with Delta = 0.1, phi^-1(0) = 0.35 (tau2^-1(0) = Delta + 1/4);
    tau2 hits the poles -1/2 at Delta and +1/2 at 1/2 + Delta (clipped to -/+6); phi diverges
    monotonically to -inf as y decreases to Delta."""
    d = 0.1
    assert abs(fe.tau2(np.array([0.35]), d)[0]) < 1e-15 and fe.tau1(np.array([0.0]))[0] == 0.0
    assert fe.tau2(np.array([d]), d)[0] == -0.5 and fe.tau2(np.array([0.5 + d]), d)[0] == 0.5
    assert fe.theta_map("phi_delta", np.array([d, 0.5 + d]), d).tolist() == [-6.0, 6.0]
    eps = np.array([1e-2, 1e-4, 1e-6, 1e-9])
    v = fe.tau1(fe.tau2(d + eps, d))
    assert np.all(np.diff(v) < 0) and v[-1] < -5.8            # Phi^-1(2e-9) = -5.88


def test_phi_delta_symmetry_and_inversion_method():
    """tau2 is a tent with its maximum at 1/2 + Delta: tau2(1/2 + Delta - t) = tau2(1/2 + Delta + t);
    the inversion method: uniform samples pushed through phi_Delta are N(0, 1)
    (Kolmogorov-Smirnov statistic < 0.01 on 10^6 samples)."""
    d = 1.0 / (4 * 2017)
    t = np.linspace(0.0, 0.5, 101)
    a = fe.tau2(np.mod(0.5 + d - t, 1.0), d)
    b = fe.tau2(np.mod(0.5 + d + t, 1.0), d)
    assert np.abs(a - b).max() < 1e-12
    y = np.random.default_rng(0).random(1_000_000)
    v = np.sort(fe.tau1(fe.tau2(y, d)))
    import scipy.stats
    ks = np.max(np.abs(scipy.stats.norm.cdf(v) - (np.arange(1, v.size + 1) / v.size)))
    assert ks < 0.01


def test_global_delta_is_the_lemma_optimum():
    """Lemma P:847-870: for prime M and a rank-1 lattice with some z_j != 0 mod M, the smaller of the
    distances of the nodes to Delta and to Delta + 1/2 is maximal at Delta = 1/(4M), where it
    equals 1/(4M) (brute force over a Delta grid on (0, 1/(2M)))."""
    from oracle import lattice
    M, z = 97, [[5, 11, 0]]
    Y = lattice.nodes(M, z, np.zeros(3), 3)
    def score(dl):
        return min(np.abs(Y - dl).min(), np.abs(Y - (dl + 0.5)).min())
    grid = np.linspace(1e-6, 1.0 / (2 * M) - 1e-6, 2001)
    best = grid[np.argmax([score(g) for g in grid])]
    assert abs(best - fe.global_delta(M)) < 1.0 / (2 * M) / 1000
    assert abs(score(fe.global_delta(M)) - 1.0 / (4 * M)) < 1e-15


# ---- the paper's example models (Sec. 4.2-4.4; Z28) --------------------------------
EX = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def test_affine_table3_indices():
    """m1(j), m2(j), k(j) of the affine example equal Table 3, and psi_j of the
    "cos_diag" family is cos(2 pi m1 x1) cos(2 pi m2 x2) with those integers: at x1 = 1/2 its
    sign is (-1)^m1 and at x2 = 1/2 it is (-1)^m2 (at x = 0 it is 1)."""
    t = EX["table3"]
    got = [fe.diag_index(j) for j in t["j"]]
    assert [g[0] for g in got] == t["m1"] and [g[1] for g in got] == t["m2"] and [g[2] for g in got] == t["k"]
    m = dict(d=20, psi="cos_diag")
    for j, m1, m2 in zip(t["j"], t["m1"], t["m2"]):
        assert fe.psi(m, j, np.array([0.0]), np.array([0.0]))[0] == 1.0
        assert abs(fe.psi(m, j, np.array([0.5]), np.array([0.0]))[0] - (-1.0) ** m1) < 1e-14
        assert abs(fe.psi(m, j, np.array([0.0]), np.array([0.5]))[0] - (-1.0) ** m2) < 1e-14
    # the diagonal enumeration covers every (m1, m2) with m1 + m2 = k exactly once per k
    for k in range(1, 12):
        js = [j for j in range(1, 200) if fe.diag_index(j)[2] == k]
        assert sorted(fe.diag_index(j)[0] for j in js) == list(range(k + 1))


def test_affine_example_bounds():
    """Affine example: c = 0.9 / zeta(2) ~ 0.547 and a_min / a_max = 1 -/+ c zeta(2)
    = 0.1 / 1.9; the preset's d = 20 coefficient stays inside them and reaches its own d-term
    extremes 1 -/+ sum amp_j at x = 0 (all psi_j = 1) for y = 0 / y = 1/2 (tent: -1 / +1)."""
    ex = EX["affine_bounds"]
    m = config("affine_example")
    c = m["amp"][0]
    assert abs(c - ex["c_printed"]) <= ex["c_tol"]
    z2 = scipy.special.zeta(ex["mu"])
    assert abs(1 - c * z2 - ex["a_min"]) < 1e-12 and abs(1 + c * z2 - ex["a_max"]) < 1e-12
    x0 = np.zeros(1)
    assert abs(fe.coefficient(m, np.zeros(20), x0, x0)[0] - (1 - sum(m["amp"]))) < 1e-14
    assert abs(fe.coefficient(m, np.full(20, 0.5), x0, x0)[0] - (1 + sum(m["amp"]))) < 1e-14
    rng = np.random.default_rng(3)
    for _ in range(30):
        a = fe.coefficient(m, rng.random(20), *rng.random((2, 300)))
        assert a.min() > ex["a_min"] and a.max() < ex["a_max"]


def test_lognormal_example_b_range():
    """Lognormal example: b(x, y) = sum_j (1/j) y_j psi_j(x) lies in [-3, 3] with
    probability > 99% for each x (y ~ N(0, I), d = 10).  b is Gaussian with variance
    sum_j (b_j(x))^2, b_j(x) = log a(x, y = e_j-probit) read through the oracle's own
    coefficient (theta = probit, y_j = Phi(1), others 1/2 -> theta = e_j); the bound must hold at
    the worst node of a fine grid, and fails if the amplitudes 1/j are dropped."""
    ex = EX["lognormal_b_range"]
    m = dict(config("lognormal_example"), theta="probit")
    d = ex["d"]
    g = np.linspace(0.0, 1.0, 401)
    x1, x2 = (v.reshape(-1) for v in np.meshgrid(g, g))
    var = np.zeros_like(x1)
    for j in range(d):
        y = np.full(d, 0.5)
        y[j] = scipy.special.ndtr(1.0)
        var += np.log(fe.coefficient(m, y, x1, x2)) ** 2
    prob = 2 * scipy.special.ndtr(ex["bound"] / np.sqrt(var.max())) - 1
    assert prob > ex["prob"]
    m1 = dict(m, amp=[1.0] * d)
    var1 = sum(np.log(fe.coefficient(m1, np.where(np.arange(d) == j, scipy.special.ndtr(1.0), 0.5),
                                     x1, x2)) ** 2 for j in range(d))
    assert 2 * scipy.special.ndtr(ex["bound"] / np.sqrt(var1.max())) - 1 < ex["prob"]


def test_lognormal_example_psi_and_f():
    """psi_j = sin(2 pi j x1) cos(2 pi (d+1-j) x2): zero on x1 = 0 and x1 = 1/2,
    separable with its x1 factor vanishing exactly at multiples of 1/(2j), and at x1 = 1/(4j),
    x2 = 0 equal to 1; f by the product-to-sum identity equals
    (sin(5.6 pi x1 + 0.3 pi x2) + sin(-3 pi x1 + 6.5 pi x2)) / 2."""
    m = config("lognormal_example")
    d = m["d"]
    for j in range(1, d + 1):
        x2 = np.linspace(0, 1, 7)
        assert np.abs(fe.psi(m, j, np.zeros(7), x2)).max() == 0.0
        assert np.abs(fe.psi(m, j, np.full(7, 0.5), x2)).max() < 1e-14
        assert abs(fe.psi(m, j, np.array([1 / (4 * j)]), np.array([0.0]))[0] - 1.0) < 1e-14
        # x2 frequency d + 1 - j: psi vanishes at x2 = 1/(4 (d+1-j))
        assert abs(fe.psi(m, j, np.array([1 / (4 * j)]), np.array([1 / (4 * (d + 1 - j))]))[0]) < 1e-14
    x1, x2 = np.random.default_rng(9).random((2, 100))
    want = 0.5 * (np.sin(5.6 * np.pi * x1 + 0.3 * np.pi * x2) + np.sin(-3.0 * np.pi * x1 + 6.5 * np.pi * x2))
    assert np.abs(fe.f_values(m, x1, x2) - want).max() < 1e-14


def test_constant_load_and_example_solves():
    """f = 1 (affine example): the centroid load is h^2 at every interior node (the six
    triangles around a node have total area 3 h^2, one third each); every example preset
    assembles to an SPD system (Cholesky succeeds) and solves to round-off; f >= 0 gives u >= 0."""
    for name in ("periodic_mu1.2", "periodic_mu3.6", "affine_example", "lognormal_example"):
        m = dict(config(name), n=12)
        if m["theta"] == "phi_delta":
            m["delta"] = fe.global_delta(101)
        cx, cy = fe.centroids(12)
        _, b = fe.assemble(12, np.ones_like(cx), fe.f_values(m, cx, cy))
        if m["f"] == "one":
            assert np.allclose(b, 1.0 / 144, rtol=1e-14, atol=0)
        rng = np.random.default_rng(5)
        for _ in range(2):
            u, rr = fe.solve(m, rng.random(m["d"]), return_residual=True)
            assert rr < 1e-11
            if m["f"] != "trig":
                assert np.all(u >= 0.0)
