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


def config(k: int, **overrides) -> dict:
    c = dict(CONFIGS[k])
    c["amp"] = list(c["amp"])
    c.update(overrides)
    return c
