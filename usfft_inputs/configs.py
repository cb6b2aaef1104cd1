"""The five workloads of BASELINE.json ``configs`` as plain data.

Each preset has a PDE model (grid n, parameter dimension d, amplitudes amp_j, the map theta,
the form of a, the right-hand side) and the detection parameters of Alg. 1 (search box
[-N, N]^d, sparsity s = s_local, r = 5 rounds (Table 2), relative threshold
1e-6 of max|c| (BASELINE; Z5), seed, and the Algorithm-A mode (Z1)).
"""
from __future__ import annotations


def _amp(c: float, d: int) -> list[float]:
    return [c / float(j * j) for j in range(1, d + 1)]          # c * j^-2


CONFIGS = {
    1: dict(name="tiny_periodic", n=16, d=4, amp=_amp(0.4, 4), theta="sin", form="affine",
            f="x2", N=8, s=20, s_local=20, r=5, theta_rel=1e-6, theta_abs=0.0, seed=0, mode="R"),
    2: dict(name="periodic_d10", n=32, d=10, amp=_amp(0.4, 10), theta="sin", form="affine",
            f="x2", N=32, s=100, s_local=100, r=5, theta_rel=1e-6, theta_abs=0.0, seed=1, mode="A"),
    3: dict(name="affine_d20", n=64, d=20, amp=_amp(0.5, 20), theta="sin", form="affine",
            f="x2", N=64, s=500, s_local=500, r=5, theta_rel=1e-6, theta_abs=0.0, seed=2, mode="A"),
    4: dict(name="lognormal_d20", n=64, d=20, amp=_amp(0.5, 20), theta="probit", form="exp",
            f="x2", N=64, s=500, s_local=500, r=5, theta_rel=1e-6, theta_abs=0.0, seed=3, mode="A"),
    5: dict(name="scale_periodic_d30", n=128, d=30, amp=_amp(0.4, 30), theta="sin", form="affine",
            f="x2", N=64, s=1000, s_local=1000, r=5, theta_rel=1e-6, theta_abs=0.0, seed=4, mode="A",
            n_test=100000),
}


# The paper's own example models (Sec. 4.2-4.4) as further workload presets (DESIGN.md §3 Z28):
# the paper's coefficient families, right-hand sides and parameter distributions on the uniform
# n = 32 mesh (G = 961 interior nodes; the paper's unstructured mesh has G = 737), with
# the detection parameters eta = I of Table 2 (N = 32, s = s_local = 100, r = 5, absolute
# threshold 1e-12).
def _amp_mu(c: float, mu: float, d: int, scale: float = 1.0) -> list[float]:
    return [scale * c * float(j) ** -mu for j in range(1, d + 1)]


_ETA_I = dict(N=32, s=100, s_local=100, r=5, theta_rel=0.0, theta_abs=1e-12, mode="A")
EXAMPLES = {
    # periodic example: a = 1 + (1/sqrt 6) sum_j sin(2 pi y_j) c j^-mu sin sin, f = x2
    "periodic_mu1.2": dict(name="periodic_mu1.2", n=32, d=10, psi="sinsin", theta="sin", form="affine",
                           f="x2", amp=_amp_mu(0.4, 1.2, 10, 6 ** -0.5), seed=11, **_ETA_I),
    "periodic_mu3.6": dict(name="periodic_mu3.6", n=32, d=10, psi="sinsin", theta="sin", form="affine",
                           f="x2", amp=_amp_mu(1.5, 3.6, 10, 6 ** -0.5), seed=12, **_ETA_I),
    # affine example: y uniform on [-1, 1] through the tent map, c = 0.9 / zeta(2),
    # mu = 2, psi_j = c j^-2 cos(2 pi m1(j) x1) cos(2 pi m2(j) x2), f = 1, d = 20
    "affine_example": dict(name="affine_example", n=32, d=20, psi="cos_diag", theta="tent", form="affine",
                           f="one", amp=_amp_mu(0.9 * 6.0 / 3.141592653589793 ** 2, 2.0, 20), seed=13,
                           **_ETA_I),
    # lognormal example: a = exp(sum_j (1/j) y_j sin(2 pi j x1) cos(2 pi (d+1-j) x2)),
    # y ~ N(0, I) through phi_Delta (Z27), f = sin(1.3 pi x1 + 3.4 pi x2) cos(4.3 pi x1 - 3.1 pi x2)
    "lognormal_example": dict(name="lognormal_example", n=32, d=10, psi="sin_cos_rev", theta="phi_delta",
                              form="exp", f="trig", amp=_amp_mu(1.0, 1.0, 10), seed=14, **_ETA_I),
}


def config(k, **overrides) -> dict:
    """BASELINE config k (1-5) or a paper example preset by name (EXAMPLES)."""
    c = dict(CONFIGS[k] if isinstance(k, int) else EXAMPLES[k])
    c["amp"] = list(c["amp"])
    c.update(overrides)
    return c
