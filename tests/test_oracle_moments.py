"""Pins of oracle/moments.py (expectation P:936-998, variance / GSI P:914-928) against what the
mathematics fixes: the expectation of known functions of uniform / normal variables computed
through the paper's periodizations and an FFT of the periodized function, Parseval, and the
ANOVA (Sobol) decomposition by brute-force conditional means."""
import itertools
import math

import numpy as np
import pytest

from oracle import fe, moments


def _coeffs_1d(fun, kind, delta=0.0, npts=1 << 16):
    """Fourier coefficients of the periodized 1-D function u(phi(x)) from an FFT on npts points."""
    x = np.arange(npts) / npts
    y = fe.theta_map(kind, x, delta)
    c = np.fft.fft(fun(y)) / npts
    k = np.fft.fftfreq(npts, 1.0 / npts).astype(np.int64)
    return k, c


@pytest.mark.parametrize("fun,want", [(lambda y: y * y, 1.0 / 3.0), (lambda y: y, 0.0),
                                      (np.exp, math.sinh(1.0))])
def test_tent_expectation_of_uniform(fun, want):
    """Y uniform on [-1, 1] (affine example): E[u(Y)] through the tent periodization and
    the D_k weights of eq. affine_ew on the FFT coefficients of u o tent."""
    k, c = _coeffs_1d(fun, "tent")
    keep = np.abs(k) <= 4000
    e = moments.expectation(k[keep, None], c[None, keep], "tent")[0]
    assert abs(e.real - want) < 2e-4 and abs(e.imag) < 1e-12


@pytest.mark.parametrize("fun,want", [(lambda y: y * y, 1.0), (lambda y: y, 0.0),
                                      (lambda y: np.exp(0.5 * y), math.exp(0.125))])
def test_phi_delta_expectation_of_normal(fun, want):
    """Y ~ N(0, 1) (lognormal example): E[u(Y)] through phi_Delta and D_{k,Delta}
     on the FFT coefficients of u o phi_Delta, for Delta = 1/(4 * 401) (Z27)."""
    delta = fe.global_delta(401)
    k, c = _coeffs_1d(fun, "phi_delta", delta, npts=1 << 18)
    keep = np.abs(k) <= 20000
    e = moments.expectation(k[keep, None], c[None, keep], "phi_delta", delta)[0]
    assert abs(e.real - want) < 5e-3 and abs(e.imag) < 1e-10


def test_tent_expectation_product_2d():
    """A 2-D product u = y1^2 exp(y2) of independent uniforms on [-1, 1]: E = (1/3) sinh(1)."""
    n = 512
    x = np.arange(n) / n
    t = fe.theta_map("tent", x)
    U = (t[:, None] ** 2) * np.exp(t[None, :])
    C = np.fft.fft2(U) / (n * n)
    k = np.fft.fftfreq(n, 1.0 / n).astype(np.int64)
    K1, K2 = np.meshgrid(k, k, indexing="ij")
    I = np.stack([K1.ravel(), K2.ravel()], 1)
    e = moments.expectation(I, C.ravel()[None, :], "tent")[0]
    assert abs(e.real - math.sinh(1.0) / 3.0) < 2e-3


def test_periodic_expectation_is_c0():
    """Periodic model: E over uniform y equals the zeroth coefficient; for
    u = sin^2(2 pi y1) cos^2(2 pi y2) that is 1/4 (and D_k = 0 for every k != 0)."""
    n = 16
    x = np.arange(n) / n
    U = np.sin(2 * np.pi * x)[:, None] ** 2 * np.cos(2 * np.pi * x)[None, :] ** 2
    C = np.fft.fft2(U) / (n * n)
    k = np.fft.fftfreq(n, 1.0 / n).astype(np.int64)
    K1, K2 = np.meshgrid(k, k, indexing="ij")
    I = np.stack([K1.ravel(), K2.ravel()], 1)
    e = moments.expectation(I, C.ravel()[None, :], "sin")[0]
    assert abs(e - 0.25) < 1e-15
    w = moments.d_weights(I, "sin")
    assert w[(I == 0).all(1)].tolist() == [1.0] and not w[~(I == 0).all(1)].any()


def _anova_by_conditional_means(F):
    """Sobol / ANOVA decomposition of a function on a full tensor grid (F has one axis per
    variable): variance of the order-l components, by inclusion-exclusion of conditional means."""
    d = F.ndim
    mean = F.mean()
    comp = {}
    for r in range(1, d + 1):
        for u in itertools.combinations(range(d), r):
            other = tuple(a for a in range(d) if a not in u)
            g = F.mean(axis=other, keepdims=True) if other else F.copy()
            for r2 in range(0, r):
                for v in itertools.combinations(u, r2):
                    g = g - (comp[v] if v else mean)
            comp[u] = g
    var_l = np.zeros(d)
    for u, g in comp.items():
        var_l[len(u) - 1] += np.mean(np.broadcast_to(g, F.shape) ** 2)
    return var_l, F.var()


def test_variance_and_gsi_match_anova():
    """sigma^2 = sum_{k != 0} |c_k|^2 equals the grid variance (Parseval), and rho(J_l) equals the
    share of the order-l Sobol components computed by conditional means, for a random
    real trigonometric polynomial in d = 3 on an 8^3 grid; sum_l rho(J_l) = 1."""
    rng = np.random.default_rng(4)
    d, n = 3, 8
    freqs = {(0, 0, 0)}
    while len(freqs) < 12:
        freqs.add(tuple(int(v) for v in rng.integers(-2, 3, size=d) * (rng.random(d) < 0.6)))
    x = np.arange(n) / n
    Y = np.meshgrid(x, x, x, indexing="ij")
    F = np.zeros((n, n, n))
    for kk in freqs:
        a, b = rng.standard_normal(2)
        F += a * np.cos(2 * np.pi * sum(kj * y for kj, y in zip(kk, Y))) + b * np.sin(
            2 * np.pi * sum(kj * y for kj, y in zip(kk, Y)))
    C = np.fft.fftn(F) / n ** 3
    k = np.fft.fftfreq(n, 1.0 / n).astype(np.int64)
    I = np.stack([a.ravel() for a in np.meshgrid(k, k, k, indexing="ij")], 1)
    var_l, var = _anova_by_conditional_means(F)
    v = moments.variance(I, C.ravel()[None, :])[0]
    rho = moments.gsi(I, C.ravel()[None, :])[0]
    assert abs(v - var) < 1e-12 * var
    assert np.allclose(rho, var_l / var, rtol=0, atol=1e-12)
    assert abs(rho.sum() - 1.0) < 1e-12


def test_gsi_single_variable_and_constant():
    """A function of y2 alone has rho(J_1) = 1; a constant has sigma^2 = 0 and rho = 0 (Z30)."""
    I = np.array([[0, 0], [0, 1], [0, -1], [0, 3]])
    C = np.array([[1.0, 0.5j, -0.5j, 0.25], [2.0, 0.0, 0.0, 0.0]])
    rho = moments.gsi(I, C)
    assert rho[0].tolist() == [1.0, 0.0] and rho[1].tolist() == [0.0, 0.0]
    assert moments.variance(I, C).tolist() == [0.5625, 0.0]


def test_d_factor_table():
    """The D_{k_j} table: 1 at 0, 0 at even k_j != 0, 2i/(pi k_j) at odd k_j;
    |D_{k_j,Delta}| = |D_{k_j}| with the phase 2 pi k_j Delta."""
    assert moments.d_factor("tent", 0) == 1 and moments.d_factor("tent", 4) == 0
    assert abs(moments.d_factor("tent", 3) - 2j / (3 * np.pi)) < 1e-16
    assert abs(moments.d_factor("tent", -1) + 2j / np.pi) < 1e-16
    z = moments.d_factor("phi_delta", 5, 0.01)
    assert abs(abs(z) - 2 / (5 * np.pi)) < 1e-16
    assert abs(np.angle(z / (2j / (5 * np.pi))) - 2 * np.pi * 5 * 0.01) < 1e-13


@pytest.mark.parametrize("kind,delta", [("tent", 0.0), ("phi_delta", 0.0123)])
def test_expectation_is_the_half_period_integral(kind, delta):
    """For an approximant that is not symmetric on the torus, sum_k c_k D_k is the integral of
    u(phi^-1(y)) against the density, i.e. 2 int_Delta^{1/2+Delta} of the trigonometric
    polynomial over the branch of phi^-1, computed here by Gauss-Legendre
    quadrature of the polynomial itself."""
    rng = np.random.default_rng(8)
    I = np.array([[k] for k in range(-7, 8)])
    C = rng.standard_normal((1, 15)) + 1j * rng.standard_normal((1, 15))
    xg, wg = np.polynomial.legendre.leggauss(64)
    x = delta + 0.25 * (xg + 1.0)                              # [Delta, 1/2 + Delta]
    u = (C @ np.exp(2j * np.pi * I @ x[None, :]))[0]
    want = 2.0 * 0.25 * np.sum(wg * u)
    got = moments.expectation(I, C, kind, delta)[0]
    assert abs(got - want) < 1e-13 * np.abs(C).sum()
