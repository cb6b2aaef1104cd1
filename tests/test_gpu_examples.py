"""GPU parity of the paper's three example models (Sec. 4.2-4.4; DESIGN.md §3 Z28) as black boxes:
the psi families (sin sin, Table 3 cos cos, sin cos reversed), the loads f = x2 / 1 / trig and
the maps sin / tent / phi_Delta, through every PCG kernel (multigrid n = 16, 32 and the scratch-slab
multigrid at n = 64; register Jacobi n = 16, 32; shared-memory Jacobi; the generic kernel at n = 20),
against the oracle's element
assembly + banded Cholesky (oracle/fe.py) on the same lattice nodes.

Tolerance: <= 1e-10 of max |u| (CG relres 1e-12 vs a direct solve).
"""
import numpy as np
import pytest
import torch

from oracle import fe as ofe
from oracle import lattice as olat
from oracle import plan as oplan
from usfft_inputs import EXAMPLES, config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2109_04131_b200 import binding
    return binding


@pytest.fixture(scope="module")
def ctx(B):
    return B.Context(0)


def _solve(B, ctx, cfg, p, b0, nb, precond, delta):
    G = (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    it = torch.empty(nb, dtype=torch.int32, device="cuda")
    rel = torch.empty(nb, dtype=torch.float64, device="cuda")
    nc = B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond=precond, delta=delta), p, b0, nb, u, nb, None,
                            it, rel, check_conv=True)
    assert nc == 0
    assert rel.max().item() <= 1e-12
    return u.cpu().numpy(), it.cpu().numpy()


@pytest.mark.parametrize("name", sorted(EXAMPLES))
@pytest.mark.parametrize("n", [32, 16, 20, 64])
def test_example_samples_every_solver(B, ctx, name, n):
    cfg = config(name, n=n)
    d, t = cfg["d"], 4
    delta = ofe.global_delta(oplan.lattice_size(cfg["s_local"], cfg["N"])) if cfg["theta"] == "phi_delta" else 0.0
    ocfg = dict(cfg, delta=delta)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, t, 1, d, cfg["N"], cfg["s"], "A", 300)
    b0, nb = 7, 21                                    # includes a ragged tail of the CTA grid
    Y = olat.nodes(p.M, p.z, p.shift, t)[:, b0:b0 + nb]
    ref = ofe.sample_pde(ocfg, Y)
    for precond in ("jacobi", "mg") if n != 20 else ("jacobi",):
        got, it = _solve(B, ctx, cfg, p, b0, nb, precond, delta)
        err = np.abs(got - ref).max() / np.abs(ref).max()
        assert err <= 1e-10, (precond, err)
        if precond == "mg":                           # high-contrast exp fields take more
            assert it.max() <= (40 if cfg["form"] == "affine" else 80)


def test_example_loads_and_nonnegativity(B, ctx):
    """f = 1 and f = x2 are >= 0, so the solutions are >= 0 (M-matrix); the trig load changes sign
    and so does u.  The f = 1 solution at a = 1 (y with theta = 0: affine example at y = 1/4,
    tent(1/4) = 0) is the discrete Poisson solution: symmetric under x1 <-> x2 and x1 <-> 1 - x1."""
    cfg = config("affine_example")
    n = cfg["n"]
    nodes = torch.full((cfg["d"], 3), 0.25, dtype=torch.float64, device="cuda")
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 2, 1, cfg["d"], cfg["N"], cfg["s"], "A", 300)
    G = (n - 1) ** 2
    u = torch.empty((G, 3), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 0, 3, u, 3, nodes)
    U = u[:, 0].cpu().numpy().reshape(n - 1, n - 1)             # [j][i]
    assert (U > 0).all()
    assert np.abs(U - U.T).max() <= 1e-12 * U.max()
    assert np.abs(U - U[:, ::-1]).max() <= 1e-12 * U.max()
    ref = ofe.solve(dict(cfg, a_func=lambda x1, x2: np.ones_like(x1)), np.zeros(cfg["d"]))
    assert np.abs(u[:, 0].cpu().numpy() - ref).max() <= 1e-11 * ref.max()
    lg = config("lognormal_example")
    M0 = oplan.lattice_size(lg["s_local"], lg["N"])
    pl = B.usfft_plan_round(ctx, lg["seed"], 2, 3, 1, lg["d"], lg["N"], lg["s"], "A", 300)
    v = torch.empty((G, 8), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(lg, delta=ofe.global_delta(M0)), pl, 0, 8, v, 8)
    V = v.cpu().numpy()
    assert (V > 0).any() and (V < 0).any()


@pytest.mark.parametrize("name", ["affine_example", "lognormal_example"])
def test_example_detector_round_trip(B, name):
    """The Detector runs the example end to end on a small box (N = 6, s = 20, n = 16): every
    sample it draws converges, I contains 0 and is symmetric under k -> -k up to the threshold
    (real-valued u), and Step 3 + the error metric run on it."""
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import uniform_points
    cfg = config(name, n=16, N=6, s=20, s_local=20)
    det = Detector(cfg)
    I, _ = det.run([])
    Ih = I.cpu().numpy().astype(np.int64)
    assert (Ih == 0).all(axis=1).any()
    cov, coef = det.step3(I)
    Y = torch.as_tensor(uniform_points(5, cfg["d"], 200), dtype=torch.float64, device="cuda")
    err, U = det.errors(I, coef, Y)
    e = err.cpu().numpy()
    assert np.isfinite(e).all() and e[:, 1].max() < 0.5 * np.abs(U.cpu().numpy()).max()
