"""GPU parity of Step 3 (reading Z26) and the accuracy metric against the
oracle (oracle/cover.py, oracle/fe.py, oracle/evaluate.py) on the same seeded inputs.

Tolerances: the cover (M, z, assignment, bins) bit-exact; coefficients of
polynomials supported on I <= 1e-12 (exact recovery); coefficients of PDE samples <= 1e-9 of
max |c| (CG relres 1e-12 vs banded Cholesky, propagated); errors <= 1e-9 relative.
"""
import numpy as np
import pytest
import torch

from oracle import cover as ocov
from oracle import evaluate as oeval
from oracle import fe as ofe
from usfft_inputs import config, trig_poly, uniform_points

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


def _set(seed, n, d, N):
    rng = np.random.default_rng(seed)
    out, seen = [], set()
    while len(out) < n:
        k = tuple(int(v) for v in rng.integers(-N, N + 1, size=d) * (rng.random(d) < 0.5))
        if k not in seen:
            seen.add(k)
            out.append(k)
    return np.array(out, dtype=np.int64)


@pytest.mark.parametrize("seed,n,d,N", [(1, 1, 3, 4), (2, 57, 4, 8), (3, 309, 10, 32), (4, 1200, 20, 64)])
def test_cover_plan_bitexact(B, ctx, seed, n, d, N):
    I = _set(seed, n, d, N)
    cov = B.usfft_cover_plan(ctx, seed, N, I)
    lat, assign, binv = ocov.build_cover(I, seed, N)
    assert cov.M == lat[0][0] and cov.z.tolist() == [z for _, z in lat]
    assert cov.assign.tolist() == assign.tolist() and cov.bin.tolist() == binv.tolist()


def _tp_blackbox(tp):
    from paper_2109_04131_b200 import binding

    def bb(det, plan, b0, nb):
        nodes = torch.empty((plan.d, nb), dtype=torch.float64, device="cuda")
        binding.usfft_lattice(det.ctx, plan, b0, nb, nodes)
        return torch.as_tensor(tp(nodes.cpu().numpy()), dtype=torch.float64, device="cuda").contiguous()
    return bb


def test_step3_exact_on_supported_polynomials(B):
    """Step 3 on a black box supported on I returns its coefficients and the oracle's."""
    from paper_2109_04131_b200.driver import Detector
    d, N, G = 5, 12, 3
    tp = trig_poly(31, d, N, G, 61, real=True, max_active=3)
    cfg = dict(d=d, N=N, s=20, s_local=20, r=1, seed=31, G=G)
    det = Detector(cfg, blackbox=_tp_blackbox(tp))
    I = torch.as_tensor(tp.freqs, dtype=torch.int16, device="cuda")
    cov, coef = det.step3(I)
    c = coef.cpu().numpy()
    c = c[..., 0] + 1j * c[..., 1]
    assert np.abs(c - tp.coefs).max() <= 1e-12
    lat, assign, binv = ocov.build_cover(tp.freqs, 31, N)
    ref, n_samples = ocov.cover_coefficients(tp, tp.freqs, lat, assign, binv)
    assert np.abs(c - ref).max() <= 1e-12
    assert n_samples == cov.M * cov.z.shape[0]


def test_step3_pde_config1_and_errors(B):
    """Config 1 (n = 16, d = 4): Step 3 on the PDE black box for a fixed frequency set, then the
    accuracy metric at 300 uniform test points, both against the oracle (FE by banded Cholesky)."""
    from paper_2109_04131_b200.driver import Detector
    cfg = config(1)
    d, N = cfg["d"], cfg["N"]
    I = _set(7, 40, d, N)
    det = Detector(cfg)
    cov, coef = det.step3(torch.as_tensor(I, dtype=torch.int16, device="cuda"))
    c = coef.cpu().numpy()
    c = c[..., 0] + 1j * c[..., 1]
    lat, assign, binv = ocov.build_cover(I, cfg["seed"], N)
    ref, _ = ocov.cover_coefficients(lambda Y: ofe.sample_pde(cfg, Y), I, lat, assign, binv)
    assert np.abs(c - ref).max() <= 1e-9 * np.abs(ref).max()
    Y = uniform_points(77, d, 300)
    err, U = det.errors(torch.as_tensor(I, dtype=torch.int16, device="cuda"), coef,
                        torch.as_tensor(Y, dtype=torch.float64, device="cuda"))
    Uo = ofe.sample_pde(cfg, Y)
    assert np.abs(U.cpu().numpy() - Uo).max() <= 1e-10 * np.abs(Uo).max()
    eo = ocov.errors(Uo, oeval.evaluate(I, ref, Y))
    assert np.abs(err.cpu().numpy() - eo).max() <= 1e-9 * eo.max()


def test_eval_err_closed_form(B, ctx):
    """usfft_eval_err on C = 0: the errors are those of Uref itself (mean |.|, rms, max)."""
    rng = np.random.default_rng(5)
    d, G, n, nI = 3, 70, 1000, 5
    I = torch.as_tensor(rng.integers(-3, 4, size=(nI, d)), dtype=torch.int16, device="cuda")
    C = torch.zeros((G, nI, 2), dtype=torch.float64, device="cuda")
    Y = torch.as_tensor(rng.random((d, n)), dtype=torch.float64, device="cuda")
    U = rng.standard_normal((G, n))
    err = torch.empty((G, 3), dtype=torch.float64, device="cuda")
    B.usfft_eval_err(ctx, I, C, Y, torch.as_tensor(U, device="cuda"), err)
    A = np.abs(U)
    want = np.stack([A.mean(1), np.sqrt((A * A).mean(1)), A.max(1)], 1)
    assert np.abs(err.cpu().numpy() - want).max() <= 1e-13 * want.max()


@pytest.mark.parametrize("cfgid", [1, 2])
def test_phi_delta_samples(B, ctx, cfgid):
    """NEXT #2 (Z27): the lognormal periodization phi_Delta as the coefficient map; the product's
    global Delta (from its own plan) equals the oracle's, and the PDE samples match the oracle
    (FE by banded Cholesky) at lattice nodes that include i = 0 and the node nearest the poles."""
    from oracle import fe as ofe2
    from oracle import lattice as olat
    from oracle import plan as oplan
    from paper_2109_04131_b200.driver import Detector
    cfg = config(cfgid, theta="phi_delta", form="exp")
    det = Detector(cfg)
    M0 = oplan.lattice_size(cfg["s_local"], cfg["N"])
    assert det.delta == ofe2.global_delta(M0)
    ocfg = dict(cfg, delta=ofe2.global_delta(M0))
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 3, 1, cfg["d"], cfg["N"], cfg["s"], "A", 300)
    nb, G = 20, (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    assert B.usfft_sample_pde(ctx, det.pde, p, 0, nb, u, nb, check_conv=True) == 0
    Y = olat.nodes(p.M, p.z, p.shift, 3)[:, :nb]
    ref = ofe.sample_pde(ocfg, Y)
    assert np.abs(u.cpu().numpy() - ref).max() <= 1e-10 * np.abs(ref).max()


@pytest.mark.parametrize("G,M,n", [(70, 401, 130), (5, 17497, 300), (33, 97, 1)])
def test_lattice_dft_bins_parity(B, ctx, G, M, n):
    """Direct lattice DFT at the bins in use vs the oracle's direct DFT (exact phase index),
    and bit-identical on an emulated 3-rank slab layout."""
    from oracle import dft as odft
    from paper_2109_04131_b200.dist import bounds
    rng = np.random.default_rng(M + n)
    U = rng.standard_normal((G, M))
    b = rng.integers(0, M, size=n).astype(np.int32)
    idx = rng.permutation(n + 3)[:n].astype(np.int32)
    coef = torch.zeros((G, n + 3, 2), dtype=torch.float64, device="cuda")
    Ud = torch.as_tensor(U, device="cuda")
    B.usfft_lattice_dft_bins(ctx, M, G, Ud, [0, M], torch.as_tensor(b, device="cuda"),
                             torch.as_tensor(idx, device="cuda"), coef)
    ref = odft.lattice_dft(U, M, b)
    got = coef.cpu().numpy()[:, idx]
    assert np.abs(got[..., 0] + 1j * got[..., 1] - ref).max() <= 1e-12 * np.abs(ref).max()
    gb, sb = bounds(G, 3), bounds(M, 3)
    r = 1
    slabs = torch.cat([Ud[gb[r]:gb[r + 1], sb[q]:sb[q + 1]].reshape(-1) for q in range(3)]).contiguous()
    c2 = torch.zeros((gb[r + 1] - gb[r], n + 3, 2), dtype=torch.float64, device="cuda")
    B.usfft_lattice_dft_bins(ctx, M, gb[r + 1] - gb[r], slabs, sb, torch.as_tensor(b, device="cuda"),
                             torch.as_tensor(idx, device="cuda"), c2)
    assert torch.equal(c2, coef[gb[r]:gb[r + 1]])


def test_step3_direct_dft_path_exact(B):
    """Step 3 with every cover lattice read by the direct DFT (the path of large covers)."""
    from paper_2109_04131_b200.driver import Detector
    d, N, G = 5, 12, 3
    tp = trig_poly(32, d, N, G, 61, real=True, max_active=3)
    det = Detector(dict(d=d, N=N, s=20, s_local=20, r=1, seed=32, G=G), blackbox=_tp_blackbox(tp))
    det.FFT_MAX_M = 0
    _, coef = det.step3(torch.as_tensor(tp.freqs, dtype=torch.int16, device="cuda"))
    c = coef.cpu().numpy()
    assert np.abs(c[..., 0] + 1j * c[..., 1] - tp.coefs).max() <= 1e-12
