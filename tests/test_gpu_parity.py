"""GPU parity: every C-ABI call against the oracle on the same seeded inputs (B200, sm_100a).

Inputs come from usfft_inputs (seeded) or from each side's own plan (the plans are compared
bit-exactly first); no oracle input and no expected value comes from the CUDA path.
Tolerances: integer/index outputs bit-exact; lattice nodes bit-exact; PDE samples
<= 1e-10 max-norm relative (CG at relres 1e-12 vs banded Cholesky); spectra/values <= 1e-12
relative to the largest |value|; decisions equal outside the Z25 fragile band.
"""
import numpy as np
import pytest
import torch

from oracle import detect as odet
from oracle import dft as odft
from oracle import evaluate as oeval
from oracle import fe as ofe
from oracle import lattice as olat
from oracle import plan as oplan
from oracle import usfft as ousfft
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


def dev(a, dtype):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype, device="cuda")


def oracle_plan(seed, step, t, i, d, N, s, nJ):
    K = 2 * N + 1
    shift = oplan.shift(seed, step, t, i, d)
    if step == 1:
        return K, 1, [[1]], shift
    M = oplan.lattice_size(s, N)
    L = oplan.num_lattices(nJ)
    return M, L, oplan.z_vectors(seed, t, i, M, L), shift


# ------------------------------------------------------------------------------ a1 plan
@pytest.mark.parametrize("step,t,i,d,N,s,nJ", [(1, 3, 2, 10, 32, 100, 65), (2, 2, 1, 4, 8, 20, 105),
                                                (2, 5, 4, 10, 32, 100, 1505), (2, 30, 1, 30, 64, 1000, 23000),
                                                (2, 7, 5, 20, 64, 500, 1)])
def test_plan_bitexact(B, ctx, step, t, i, d, N, s, nJ):
    for seed in (0, 1, 4):
        p = B.usfft_plan_round(ctx, seed, step, t, i, d, N, s, "A", nJ)
        M, L, z, shift = oracle_plan(seed, step, t, i, d, N, s, nJ)
        assert (p.M, p.L) == (M, L)
        assert p.z.tolist() == [list(map(int, r)) for r in z]
        assert np.array_equal(p.shift, np.array(shift))


def test_mode_r_plan_bitexact(B, ctx):
    rng = np.random.default_rng(5)
    I_prev = rng.integers(-8, 9, size=(30, 2))
    kt = np.arange(-3, 4)
    J = olat.candidates(I_prev, kt)
    p = B.usfft_plan_round(ctx, 9, 2, 3, 2, 4, 8, 20, "R", J.shape[0], dev(I_prev, torch.int16),
                           I_prev.shape[0], dev(kt, torch.int16))
    M, z = ousfft.mode_r_lattice(J, 9, 3, 2, 8)
    assert p.M == M and p.L == 1 and p.z.tolist() == [list(map(int, r)) for r in z]


# ------------------------------------------------------------------------------ a2 + a3 lattice
def test_nodes_and_bins_bitexact(B, ctx):
    rng = np.random.default_rng(1)
    d, t = 10, 4
    p = B.usfft_plan_round(ctx, 1, 2, t, 3, d, 32, 100, "A", 1505)
    I_prev = rng.integers(-32, 33, size=(43, t - 1))
    kt = np.array([-5, 0, 3, 17, 31])
    J = olat.candidates(I_prev, kt)
    Btot = p.L * p.M
    for b0, nb in ((0, Btot), (17, Btot - 40), (Btot - 1, 1)):
        nodes = torch.empty((d, nb), dtype=torch.float64, device="cuda")
        bins = torch.empty((p.L, J.shape[0]), dtype=torch.int32, device="cuda")
        B.usfft_lattice(ctx, p, b0, nb, nodes, dev(I_prev, torch.int16), I_prev.shape[0],
                        dev(kt, torch.int16), bins)
        ref = olat.nodes(p.M, p.z, p.shift, t)[:, b0:b0 + nb]
        assert np.array_equal(nodes.cpu().numpy(), ref)
        assert np.array_equal(bins.cpu().numpy(), olat.bins(J, p.z, p.M))
    # Step-1 line lattice
    p1 = B.usfft_plan_round(ctx, 1, 1, 7, 2, d, 32, 100, "A", 65)
    nodes = torch.empty((d, 65), dtype=torch.float64, device="cuda")
    B.usfft_lattice(ctx, p1, 0, 65, nodes)
    assert np.array_equal(nodes.cpu().numpy(), olat.nodes(65, [[1]], p1.shift, 1, line_axis=6))


def test_injectivity_flag(B, ctx):
    from paper_2109_04131_b200.binding import Plan
    J = np.array([[0, 0], [1, 0], [0, 1], [5, 0]])
    p = Plan(2, 5, 2, 2, -1, np.array([[1, 2], [1, 3]]), np.zeros(2))
    Jd = dev(J[:, :1], torch.int16)
    # kt must be the last component: build J = I_prev x kt with I_prev=J[:,0] rows, kt=[0,1] -> check spec example
    inj = B.usfft_lattice(ctx, p, 0, 0, None, dev(np.array([[0], [1], [5]]), torch.int16), 3,
                          dev(np.array([0, 1]), torch.int16), None, injective=True)
    Jfull = olat.candidates(np.array([[0], [1], [5]]), np.array([0, 1]))
    want = [int(olat.injective(olat.bins(Jfull, [z], 5)[0])) for z in p.z]
    assert inj == want and inj == [0, 0]


# ------------------------------------------------------------------------------ a4 + a5 PDE
@pytest.mark.parametrize("cfgid,nb", [(1, 45), (2, 37), (3, 9), (4, 9), (5, 4)])
def test_sample_pde_parity(B, ctx, cfgid, nb):
    cfg = config(cfgid)
    t = 3
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, t, 1, cfg["d"], cfg["N"], cfg["s"], "A", 200)
    b0 = 11
    G = (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    iters = torch.empty(nb, dtype=torch.int32, device="cuda")
    rel = torch.empty(nb, dtype=torch.float64, device="cuda")
    nc = B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, b0, nb, u, nb, None, iters, rel, check_conv=True)
    assert nc == 0
    Y = olat.nodes(p.M, p.z, p.shift, t)[:, b0:b0 + nb]
    ref = ofe.sample_pde(cfg, Y)
    got = u.cpu().numpy()
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= 1e-10, err
    assert rel.max().item() <= 1e-12 and iters.min().item() > 0
    # the same samples solved as two ragged launches are bit-identical (no batch-position effects)
    u2 = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    h = nb // 3
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, b0, h, u2[:, :h].contiguous(), h)
    part = torch.empty((G, nb - h), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, b0 + h, nb - h, part, nb - h)
    first = torch.empty((G, h), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, b0, h, first, h)
    assert torch.equal(torch.cat([first, part], 1), u)


def test_sample_pde_explicit_nodes_match_fused(B, ctx):
    cfg = config(2)
    p = B.usfft_plan_round(ctx, 1, 2, 5, 2, 10, 32, 100, "A", 900)
    nb = 50
    nodes = torch.empty((10, nb), dtype=torch.float64, device="cuda")
    B.usfft_lattice(ctx, p, 100, nb, nodes)
    G = 961
    a = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    b = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 100, nb, a, nb)
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 100, nb, b, nb, nodes)
    assert torch.equal(a, b)


def test_noconv_reported(B, ctx):
    cfg = config(2)
    p = B.usfft_plan_round(ctx, 1, 2, 2, 1, 10, 32, 100, "A", 50)
    u = torch.empty((961, 8), dtype=torch.float64, device="cuda")
    nc = B.usfft_sample_pde(ctx, B.pde_desc(cfg, maxit=3), p, 0, 8, u, 8, check_conv=True)
    assert nc == 8


# ------------------------------------------------------------------------------ a7 + a8 FFT, keys
def _round_inputs(seed, G, M, L, nJ, t=3):
    rng = np.random.default_rng(seed)
    U = rng.standard_normal((G, L * M))
    z = rng.integers(1, M, size=(L, t))
    J = rng.integers(-20, 21, size=(nJ, t))
    return U, z, J, olat.bins(J, z, M)


@pytest.mark.parametrize("G,M,L,nJ", [(7, 97, 11, 130), (33, 401, 5, 777), (5, 17, 1, 17), (3, 2017, 3, 50)])
def test_lattice_fft_parity(B, ctx, G, M, L, nJ):
    from paper_2109_04131_b200.binding import Plan
    U, z, J, bins = _round_inputs(G + M, G, M, L, nJ)
    p = Plan(3, M, L, 3, -1, z, np.zeros(3))
    Mh = M // 2 + 1
    spectra = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    kmin = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
    kmax = torch.empty(1, dtype=torch.float64, device="cuda")
    Ud = dev(U, torch.float64)
    B.usfft_lattice_fft(ctx, p, G, Ud, [0, L * M], dev(bins, torch.int32), nJ, spectra, kmin, kmax)
    sp = spectra.cpu().numpy()
    ref = np.stack([odft.lattice_dft(U[:, l * M:(l + 1) * M], M, np.arange(Mh)) for l in range(L)], 1)
    got = (sp[..., 0] + 1j * sp[..., 1]) / M
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    V = odft.round_values(U, M, L, bins)
    km_ref = odet.kappa_min(V)
    km = kmin.cpu().numpy()
    assert np.abs(np.sqrt(km) - np.sqrt(km_ref)).max() <= 1e-12 * np.sqrt(km_ref.max())
    assert kmax.item() == km.max()
    # emulated 3-rank exchange: node range of rank 1 with samples in 3 slabs -> bit-identical
    P = 3
    from paper_2109_04131_b200.dist import bounds
    gb, sb = bounds(G, P), bounds(L * M, P)
    r = 1
    slabs = torch.cat([Ud[gb[r]:gb[r + 1], sb[q]:sb[q + 1]].reshape(-1) for q in range(P)])
    gl = gb[r + 1] - gb[r]
    sp2 = torch.empty((gl, L, Mh, 2), dtype=torch.float64, device="cuda")
    km2 = torch.empty((gl, nJ), dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, gl, slabs.contiguous(), sb, dev(bins, torch.int32), nJ, sp2, km2, kmax)
    assert torch.equal(sp2, spectra[gb[r]:gb[r + 1]]) and torch.equal(km2, kmin[gb[r]:gb[r + 1]])


@pytest.mark.parametrize("G,M,L,nJ", [(19, 401, 17, 1000), (9, 97, 11, 300), (4, 2017, 3, 70), (11, 401, 35, 9000)])
def test_keys_vs_oracle(B, ctx, G, M, L, nJ):
    """a8 keys of the grouped key kernel (bins tile shared by 8 nodes, G not a multiple of 8)
    against the oracle's kappa_min of the oracle's direct-DFT values; kappa_max exact."""
    from paper_2109_04131_b200.binding import Plan
    U, z, J, bins = _round_inputs(G * M, G, M, L, nJ)
    p = Plan(3, M, L, 3, -1, z, np.zeros(3))
    Mh = M // 2 + 1
    spectra = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    kmin = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
    kmax = torch.empty(1, dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, G, dev(U, torch.float64), [0, L * M], dev(bins, torch.int32), nJ, spectra,
                        kmin, kmax)
    km = kmin.cpu().numpy()
    ref = odet.kappa_min(odft.round_values(U, M, L, bins))
    assert np.abs(np.sqrt(km) - np.sqrt(ref)).max() <= 1e-12 * np.sqrt(ref.max())
    assert kmax.item() == km.max()


# ------------------------------------------------------------------------------ a9-a11 selection
@pytest.mark.parametrize("G,nJ,s", [(5, 1000, 7), (17, 4097, 100), (3, 9, 20), (4, 600, 600), (2, 1, 1)])
def test_select_union_bitexact(B, ctx, G, nJ, s):
    rng = np.random.default_rng(nJ + s)
    km = rng.choice(np.r_[0.0, rng.random(50), 1e-13, 1e-20], size=(G, nJ))   # ties + zeros
    kmax_h = km.max()
    th2_ref = odet.theta_squared(km, 1e-6)
    D, votes_ref = odet.select(km, s, th2_ref)
    kmd = dev(km, torch.float64)
    votes = torch.empty(nJ, dtype=torch.int32, device="cuda")
    det_g = torch.empty((G, s), dtype=torch.int32, device="cuda")
    ndg = torch.empty(G, dtype=torch.int32, device="cuda")
    th2 = torch.empty(1, dtype=torch.float64, device="cuda")
    B.usfft_detect_select(ctx, G, nJ, kmd, dev([kmax_h], torch.float64), s, 1e-6, 0.0, votes, det_g, ndg, th2)
    assert th2.item() == th2_ref
    assert np.array_equal(votes.cpu().numpy(), votes_ref)
    dg, nd = det_g.cpu().numpy(), ndg.cpu().numpy()
    for g in range(G):
        assert dg[g, :nd[g]].tolist() == D[g].tolist()
        assert np.all(dg[g, nd[g]:] == -1)
    flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
    flags[::5] = 1
    fl_ref = flags.cpu().numpy().astype(bool) | (votes_ref > 0)
    det_idx = torch.empty(nJ, dtype=torch.int32, device="cuda")
    uni = torch.empty(nJ, dtype=torch.int32, device="cuda")
    n_det, n_u = B.usfft_detect_union(ctx, nJ, votes, flags, det_idx, uni)
    assert det_idx[:n_det].cpu().tolist() == np.nonzero(votes_ref)[0].tolist()
    assert uni[:n_u].cpu().tolist() == np.nonzero(fl_ref)[0].tolist()
    assert np.array_equal(flags.cpu().numpy().astype(bool), fl_ref)


def test_select_all_zero_keys(B, ctx):
    G, nJ, s = 3, 50, 5
    z = torch.zeros((G, nJ), dtype=torch.float64, device="cuda")
    votes = torch.empty(nJ, dtype=torch.int32, device="cuda")
    det_g = torch.empty((G, s), dtype=torch.int32, device="cuda")
    ndg = torch.empty(G, dtype=torch.int32, device="cuda")
    B.usfft_detect_select(ctx, G, nJ, z, torch.zeros(1, dtype=torch.float64, device="cuda"), s, 1e-6, 0.0,
                          votes, det_g, ndg)
    assert votes.sum().item() == 0 and ndg.sum().item() == 0


@pytest.mark.parametrize("G,M,L,nJ,s", [(9, 97, 11, 300, 20), (6, 401, 7, 1200, 60), (4, 17, 1, 17, 5)])
def test_round_stage_parity_from_samples(B, ctx, G, M, L, nJ, s):
    """a7-a12 from the same seeded samples (a sparse trig polynomial plus noise floor):
    decisions equal outside the fragile band, resolved values <= 1e-12 of max|v|."""
    from paper_2109_04131_b200.binding import Plan
    rng = np.random.default_rng(M + nJ)
    t = 3
    z = rng.integers(1, M, size=(L, t))
    J = np.unique(rng.integers(-6, 7, size=(nJ, t)), axis=0)
    nJ = J.shape[0]
    bins = olat.bins(J, z, M)
    tp = trig_poly(int(M + nJ), t, 6, G, 24, real=True)
    Y = olat.nodes(M, z, np.zeros(t), t)
    U = tp(Y) + 1e-9 * rng.standard_normal((G, L * M))
    p = Plan(t, M, L, t, -1, z, np.zeros(t))
    Mh = M // 2 + 1
    spectra = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    kmin = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
    kmax = torch.empty(1, dtype=torch.float64, device="cuda")
    bd = dev(bins, torch.int32)
    B.usfft_lattice_fft(ctx, p, G, dev(U, torch.float64), [0, L * M], bd, nJ, spectra, kmin, kmax)
    votes = torch.empty(nJ, dtype=torch.int32, device="cuda")
    det_g = torch.empty((G, s), dtype=torch.int32, device="cuda")
    ndg = torch.empty(G, dtype=torch.int32, device="cuda")
    B.usfft_detect_select(ctx, G, nJ, kmin, kmax, s, 1e-6, 0.0, votes, det_g, ndg)
    flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
    det_idx = torch.empty(nJ, dtype=torch.int32, device="cuda")
    n_det, _ = B.usfft_detect_union(ctx, nJ, votes, flags, det_idx)
    V = odft.round_values(U, M, L, bins)
    ref = odet.detect_round(V, bins, s, 1e-6)
    frag = odet.fragile(ref["kappa_min"], s, ref["theta2"])
    dg, nd = det_g.cpu().numpy(), ndg.cpu().numpy()
    for g in range(G):                       # decisions agree except inside the Z25 band
        diff = set(dg[g, :nd[g]].tolist()) ^ set(ref["D"][g].tolist())
        assert all(frag[g, k] for k in diff)
    if frag.any():
        return
    assert det_idx[:n_det].cpu().tolist() == ref["det"].tolist()
    coef = torch.empty((G, n_det, 2), dtype=torch.float64, device="cuda")
    lstar = torch.empty((G, n_det), dtype=torch.int32, device="cuda")
    B.usfft_resolve(ctx, p, G, spectra, bd, nJ, det_g, ndg, s, det_idx, n_det, coef, lstar)
    c = coef.cpu().numpy()
    assert np.array_equal(lstar.cpu().numpy(), ref["lstar"])
    vmax = np.abs(V).max()
    assert np.abs(c[..., 0] + 1j * c[..., 1] - ref["coef"]).max() <= 1e-12 * vmax


# ------------------------------------------------------------------------------ whole Alg. 1
def _tp_blackbox(tp):
    from paper_2109_04131_b200 import binding

    def bb(det, plan, b0, nb):
        nodes = torch.empty((plan.d, nb), dtype=torch.float64, device="cuda")
        binding.usfft_lattice(det.ctx, plan, b0, nb, nodes)
        return torch.as_tensor(tp(nodes.cpu().numpy()), dtype=torch.float64, device="cuda").contiguous()
    return bb


@pytest.mark.parametrize("mode,factor", [("A", 1), ("R", 1), ("A", 3)])
def test_full_run_trig_poly_matches_oracle(B, mode, factor):
    from paper_2109_04131_b200.driver import Detector
    d, N, G = 6, 16, 4
    for trial in range(3):
        tp = trig_poly(900 + trial, d, N, G, 16, real=True, max_active=3)
        cfg = dict(d=d, N=N, s=20, s_local=20, r=5, seed=trial, theta_rel=1e-6, mode=mode, G=G,
                   lattice_factor=factor)
        det = Detector(cfg, blackbox=_tp_blackbox(tp))
        I, C = det.run()
        ref = ousfft.run(cfg, tp)
        Ig = I.cpu().numpy().astype(np.int64)
        assert Ig.tolist() == ref["I"].tolist()
        Cg = C.cpu().numpy()
        assert np.abs(Cg[..., 0] + 1j * Cg[..., 1] - ref["C"]).max() <= 1e-12
        # exact recovery of the polynomial (Thm 1.1)
        assert {tuple(k) for k in Ig.tolist()} == {tuple(k) for k in tp.freqs.tolist()}


def test_full_run_pde_config1(B):
    """Config 1 (mode A for runtime): GPU Alg. 1 vs oracle Alg. 1 on the PDE black box."""
    from paper_2109_04131_b200.driver import Detector
    from parity import compare_round
    cfg = config(1, mode="A")
    det = Detector(cfg)
    log_g = []
    I, C = det.run(log_g)
    log_o, trace = [], []
    ref = ousfft.run(cfg, lambda Y: ofe.sample_pde(cfg, Y), log_o, trace)
    assert [(e["t"], e["i"], e["M"], e.get("L", 1)) for e in log_g] == \
        [(e["t"], e["i"], e.get("M", 17), e.get("L", 1)) for e in log_o]
    Ig = I.cpu().numpy().astype(np.int64)
    assert Ig.tolist() == ref["I"].tolist()
    last, rr = det.last_round, trace[-1]
    frag = odet.fragile(rr["kappa_min"], cfg["s"], rr["theta2"])
    cm = np.abs(rr["coef"]).max()
    compare_round(last.det_g.cpu().numpy(), last.n_det_g.cpu().numpy(), last.det_idx.cpu().numpy(),
                  last.lstar.cpu().numpy(), last.coef.cpu().numpy(), rr, frag, 1e-9 * cm)


# ------------------------------------------------------------------------------ eval
def test_eval_parity(B, ctx):
    rng = np.random.default_rng(3)
    d, G, nI, n = 10, 70, 133, 1000
    I = rng.integers(-32, 33, size=(nI, d)) * (rng.random((nI, d)) < 0.3)
    Cc = rng.standard_normal((G, nI)) + 1j * rng.standard_normal((G, nI))
    Y = uniform_points(4, d, n)
    U = torch.empty((G, n), dtype=torch.float64, device="cuda")
    Cd = dev(np.stack([Cc.real, Cc.imag], -1), torch.float64)
    B.usfft_eval(ctx, dev(I, torch.int16), Cd, dev(Y, torch.float64), U)
    ref = oeval.evaluate(I, Cc, Y).real
    assert np.abs(U.cpu().numpy() - ref).max() <= 1e-11 * np.abs(Cc).sum(1).max()


# ------------------------------------------------------------------------------ kernel variants
@pytest.mark.parametrize("G,M,L", [(5, 401, 3), (2, 4001, 2), (4, 97, 5), (3, 2017, 2), (6, 61, 3),
                                    (7, 65, 2), (5, 17, 3), (3, 2, 2)])
def test_fft_paths_vs_oracle(B, ctx, G, M, L):
    """Every lattice-FFT path, each on the M that selects it: the register four-step Rader
    (M = 401), the compile-time Rader/Stockham plans (97, 2017, 4001), the runtime-plan Rader
    (61: 60 = 4 * 3 * 5) and the direct DFT (65, 17, 2: not Rader-able) against the oracle's
    direct DFT (odd L included)."""
    from paper_2109_04131_b200.binding import Plan
    U, z, J, bins = _round_inputs(M, G, M, L, 64)
    p = Plan(3, M, L, 3, -1, z, np.zeros(3))
    Mh = M // 2 + 1
    sp = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, G, dev(U, torch.float64), [0, L * M], None, 0, sp, None, None)
    o = sp.cpu().numpy()
    ref = np.stack([odft.lattice_dft(U[:, l * M:(l + 1) * M], M, np.arange(Mh)) for l in range(L)], 1) * M
    assert np.abs(o[..., 0] + 1j * o[..., 1] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_pcg_preconditioners_agree(B, ctx):
    """Multigrid-preconditioned CG (default for power-of-two meshes) and the Jacobi PCG both meet
    the oracle tolerance on the same samples."""
    for cfgid in (1, 2):
        cfg = config(cfgid)
        p = B.usfft_plan_round(ctx, cfg["seed"], 2, 4, 2, cfg["d"], cfg["N"], cfg["s"], "A", 300)
        nb, G = 24, (cfg["n"] - 1) ** 2
        Y = olat.nodes(p.M, p.z, p.shift, 4)[:, 5:5 + nb]
        ref = ofe.sample_pde(cfg, Y)
        for precond in ("mg", "jacobi"):
            u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
            it = torch.empty(nb, dtype=torch.int32, device="cuda")
            rel = torch.empty(nb, dtype=torch.float64, device="cuda")
            assert B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond=precond), p, 5, nb, u, nb, None,
                                      it, rel, check_conv=True) == 0
            assert np.abs(u.cpu().numpy() - ref).max() <= 1e-10 * np.abs(ref).max()
            assert rel.max().item() <= 1e-12
            if precond == "mg":
                assert it.max().item() <= 30           # multigrid: iteration count ~ mesh independent


def test_pcg_all_samples_of_a_round_converge(B, ctx):
    """Every sample of a full config-2 round converges (guards against NaN/stagnation paths)."""
    cfg = config(2)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 3, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
    nb, G = p.L * p.M, 961
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    iters = torch.empty(nb, dtype=torch.int32, device="cuda")
    rel = torch.empty(nb, dtype=torch.float64, device="cuda")
    assert B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 0, nb, u, nb, None, iters, rel, check_conv=True) == 0
    assert torch.isfinite(u).all() and rel.max().item() <= 1e-12
    assert iters.max().item() < 300


def test_emulated_multirank_round_bitexact(B, ctx):
    """A whole Step-2 round computed as P = 3 virtual ranks (sample shards, exchanged slabs, node
    shards, kappa_max MAX, votes SUM) is bit-identical to the P = 1 round.  The
    exchange is emulated by slicing on one GPU; the NCCL calls themselves are plumbing."""
    from paper_2109_04131_b200.dist import bounds
    cfg = config(2)
    t, s = 3, cfg["s_local"]
    rng = np.random.default_rng(12)
    I_prev = np.unique(rng.integers(-8, 9, size=(40, t - 1)), axis=0)
    kt = np.arange(-3, 4)
    Id, ktd = dev(I_prev, torch.int16), dev(kt, torch.int16)
    nJ = I_prev.shape[0] * kt.shape[0]
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, t, 2, cfg["d"], cfg["N"], s, "A", nJ)
    Bt, G, Mh = p.L * p.M, 961, p.M // 2 + 1
    bins = torch.empty((p.L, nJ), dtype=torch.int32, device="cuda")
    B.usfft_lattice(ctx, p, 0, 0, None, Id, I_prev.shape[0], ktd, bins)
    pde = B.pde_desc(cfg)

    def one_round(P):
        sb, gb = bounds(Bt, P), bounds(G, P)
        u_r = []
        for r in range(P):                                   # sample shards
            nb = sb[r + 1] - sb[r]
            u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
            B.usfft_sample_pde(ctx, pde, p, sb[r], nb, u, nb)
            u_r.append(u)
        kmaxes, kmins, specs = [], [], []
        for r in range(P):                                   # exchanged slabs -> node shards
            gl = gb[r + 1] - gb[r]
            slab = torch.cat([u_r[q][gb[r]:gb[r + 1]].reshape(-1) for q in range(P)]).contiguous()
            sp = torch.empty((gl, p.L, Mh, 2), dtype=torch.float64, device="cuda")
            km = torch.empty((gl, nJ), dtype=torch.float64, device="cuda")
            kx = torch.empty(1, dtype=torch.float64, device="cuda")
            B.usfft_lattice_fft(ctx, p, gl, slab, sb, bins, nJ, sp, km, kx)
            kmaxes.append(kx), kmins.append(km), specs.append(sp)
        kmax = torch.stack(kmaxes).max().reshape(1)          # all-reduce MAX
        votes_all = torch.zeros(nJ, dtype=torch.int32, device="cuda")
        outs = []
        for r in range(P):
            gl = gb[r + 1] - gb[r]
            v = torch.empty(nJ, dtype=torch.int32, device="cuda")
            dg_ = torch.empty((gl, s), dtype=torch.int32, device="cuda")
            nd_ = torch.empty(gl, dtype=torch.int32, device="cuda")
            B.usfft_detect_select(ctx, gl, nJ, kmins[r], kmax, s, 1e-6, 0.0, v, dg_, nd_)
            votes_all += v                                   # all-reduce SUM
            outs.append((dg_, nd_))
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        det = torch.empty(nJ, dtype=torch.int32, device="cuda")
        n_det, _ = B.usfft_detect_union(ctx, nJ, votes_all, flags, det)
        coefs = []
        for r in range(P):
            gl = gb[r + 1] - gb[r]
            cf = torch.empty((gl, n_det, 2), dtype=torch.float64, device="cuda")
            B.usfft_resolve(ctx, p, gl, specs[r], bins, nJ, outs[r][0], outs[r][1], s, det, n_det, cf)
            coefs.append(cf)
        return (torch.cat(u_r, 1), torch.cat(kmins), kmax, votes_all, det[:n_det].clone(),
                torch.cat(coefs))

    a, b = one_round(1), one_round(3)
    for x, y in zip(a, b):
        assert torch.equal(x, y)


@pytest.mark.parametrize("n", [301, 1])
def test_eval_vs_oracle(B, ctx, n):
    """usfft_eval and usfft_eval_err on the fp64 tensor pipe (DMMA) against the oracle's direct
    double sum; odd sizes exercise every tile edge."""
    rng = np.random.default_rng(8 + n)
    d, G, nI = 7, 37, 45
    I = rng.integers(-9, 10, size=(nI, d)) * (rng.random((nI, d)) < 0.4)
    Cc = rng.standard_normal((G, nI)) + 1j * rng.standard_normal((G, nI))
    Y = rng.random((d, n))
    ref = oeval.evaluate(I, Cc, Y).real
    Cd = dev(np.stack([Cc.real, Cc.imag], -1), torch.float64)
    U = torch.empty((G, n), dtype=torch.float64, device="cuda")
    B.usfft_eval(ctx, dev(I, torch.int16), Cd, dev(Y, torch.float64), U)
    assert np.abs(U.cpu().numpy() - ref).max() <= 1e-11 * np.abs(Cc).sum(1).max()
    # the accuracy metric: complex modulus errors against a reference with a known
    # offset from the approximant
    Uref = rng.standard_normal((G, n))
    err = torch.empty((G, 3), dtype=torch.float64, device="cuda")
    B.usfft_eval_err(ctx, dev(I, torch.int16), Cd, dev(Y, torch.float64), dev(Uref, torch.float64), err)
    D = np.abs(Uref - oeval.evaluate(I, Cc, Y))
    want = np.stack([D.mean(1), np.sqrt((D * D).mean(1)), D.max(1)], 1)
    assert np.abs(err.cpu().numpy() - want).max() <= 1e-11 * want.max()


@pytest.mark.parametrize("cfgid,n,nb", [(3, 64, 9), (4, 64, 7), (5, 128, 4), (1, 8, 13), (2, 16, 11)])
def test_pcg_mg_every_mesh(B, ctx, cfgid, n, nb):
    """The multigrid CG of every mesh (n = 8 .. 128) meets the oracle tolerance with a
    mesh-independent iteration count; the same samples solved in two ragged launches are
    bit-identical."""
    cfg = config(cfgid, n=n)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 3, 1, cfg["d"], cfg["N"], cfg["s"], "A", 200)
    G = (n - 1) ** 2
    Y = olat.nodes(p.M, p.z, p.shift, 3)[:, 3:3 + nb]
    ref = ofe.sample_pde(cfg, Y)
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    it = torch.empty(nb, dtype=torch.int32, device="cuda")
    rel = torch.empty(nb, dtype=torch.float64, device="cuda")
    assert B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond="mg"), p, 3, nb, u, nb, None, it, rel,
                              check_conv=True) == 0
    assert np.abs(u.cpu().numpy() - ref).max() <= 1e-10 * np.abs(ref).max()
    assert rel.max().item() <= 1e-12 and it.max().item() <= 30
    # bit-identical when the same samples are solved in two ragged launches
    h = nb // 2
    a = torch.empty((G, h), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond="mg"), p, 3, h, a, h)
    assert torch.equal(a, u[:, :h])


@pytest.mark.parametrize("d", [1, 2])
def test_full_run_low_dimensions(B, d):
    """Degenerate dimensions: d = 1 (Step 1 only, no Step-2 round) and d = 2 (one Step-2 round
    with s~ = s): the detected set equals the oracle's and the polynomial's support."""
    from paper_2109_04131_b200.driver import Detector
    N, G = 12, 3
    tp = trig_poly(950 + d, d, N, G, 7, real=True, max_active=d)
    cfg = dict(d=d, N=N, s=12, s_local=12, r=3, seed=d, theta_rel=1e-6, mode="A", G=G)
    det = Detector(cfg, blackbox=_tp_blackbox(tp))
    I, C = det.run()
    ref = ousfft.run(cfg, tp)
    Ig = I.cpu().numpy().astype(np.int64).reshape(-1, d)
    assert Ig.tolist() == np.asarray(ref["I"]).reshape(-1, d).tolist()
    assert {tuple(k) for k in Ig.tolist()} == {tuple(k) for k in tp.freqs.tolist()}
    cov, coef = det.step3(I.reshape(-1, d).contiguous())
    c = coef.cpu().numpy()
    order = {tuple(k): a for a, k in enumerate(tp.freqs.tolist())}
    want = tp.coefs[:, [order[tuple(k)] for k in Ig.tolist()]]
    assert np.abs(c[..., 0] + 1j * c[..., 1] - want).max() <= 1e-12


@pytest.mark.parametrize("G,M,L,nJ", [(3, 4001, 2, 300)])
def test_lattice_fft_largest_prime(B, ctx, G, M, L, nJ):
    """M = 4001 (config 5's Step-2 lattices, the 4000-point Rader template): spectra and keys."""
    from paper_2109_04131_b200.binding import Plan
    U, z, J, bins = _round_inputs(G + M, G, M, L, nJ)
    p = Plan(3, M, L, 3, -1, z, np.zeros(3))
    Mh = M // 2 + 1
    spectra = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    kmin = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
    kmax = torch.empty(1, dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, G, dev(U, torch.float64), [0, L * M], dev(bins, torch.int32), nJ, spectra, kmin, kmax)
    sp = spectra.cpu().numpy()
    ref = np.stack([odft.lattice_dft(U[:, l * M:(l + 1) * M], M, np.arange(Mh)) for l in range(L)], 1)
    assert np.abs((sp[..., 0] + 1j * sp[..., 1]) / M - ref).max() <= 1e-12 * np.abs(ref).max()
    km_ref = odet.kappa_min(odft.round_values(U, M, L, bins))
    assert np.abs(np.sqrt(kmin.cpu().numpy()) - np.sqrt(km_ref)).max() <= 1e-12 * np.sqrt(km_ref.max())
