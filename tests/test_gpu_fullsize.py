"""GPU parity on the full-size paths the benchmark runs (SURVEY §8(c) "scale-out").

The solver kernels loop over many samples per CTA / cluster; the FFT, key, select and resolve
kernels run on every node of a bench round.  These tests drive exactly those launches:
  * a whole Step-2 round of samples of every BASELINE config (configs 2-5: tens of thousands of
    samples, many per CTA or cluster), with the oracle's banded Cholesky on a random subset of 64;
  * one bench round per config with the oracle's direct DFT on 64 sampled nodes and the oracle's
    keys, threshold, per-node selection, union and resolve consuming the GPU's spectra of all
    nodes (GPU-fed stage parity; decisions compared per Z25 with the strict set check);
  * config 2's whole detection (Steps 1-2, 91 rounds) against the oracle's own Alg. 1 on its own
    FE solves.
The oracle's solves run in a process pool (samples are independent); nothing here feeds the
oracle from the CUDA path except where named "GPU-fed".
"""
import multiprocessing as mp
import os

import numpy as np
import pytest
import torch

from oracle import detect as odet
from oracle import dft as odft
from oracle import fe as ofe
from oracle import lattice as olat
from oracle import usfft as ousfft
from usfft_inputs import config

pytestmark = pytest.mark.gpu

# |J_t| of the round each config's bench times (t = 5; config 4 at t = 2, see below)
ROUND = {2: (5, 1000), 3: (5, 1755), 4: (3, 2031105), 5: (5, 1105)}


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2109_04131_b200 import binding
    return binding


@pytest.fixture(scope="module")
def ctx(B):
    return B.Context(0)


@pytest.fixture(scope="module")
def pool():
    p = mp.get_context("fork").Pool(max(1, min(32, os.cpu_count() or 1)))
    yield p
    p.close()


def _solve_cols(job):
    cfg, Y = job
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return ofe.sample_pde(cfg, Y)


def oracle_solves(pool, cfg, Y):
    """The oracle's FE solves of the columns of Y, spread over the pool (same results as
    ofe.sample_pde(cfg, Y): each column is one independent banded-Cholesky solve)."""
    k = max(1, min(len(pool._pool), Y.shape[1]))
    parts = np.array_split(np.arange(Y.shape[1]), k)
    outs = pool.map(_solve_cols, [(cfg, Y[:, p]) for p in parts if p.size])
    return np.concatenate(outs, axis=1)


@pytest.mark.parametrize("cfgid", [2, 3, 4, 5])
def test_sample_pde_whole_round(B, ctx, pool, cfgid):
    """All L*M samples of a bench-sized round in one call (>= 20 samples per CTA / cluster on
    the persistent loop); 64 random samples against the oracle's banded Cholesky (<= 1e-10
    max-norm relative), every sample at relres <= 1e-12 within 14 CG iterations, and a ragged re-solve of a sub-range
    bit-identical (a sample's result does not depend on its CTA, cluster or launch)."""
    cfg = config(cfgid)
    t, nJ = ROUND[cfgid]
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, t, 1, cfg["d"], cfg["N"], cfg["s_local"], "A", nJ)
    nb, G = p.L * p.M, (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    it = torch.empty(nb, dtype=torch.int32, device="cuda")
    rel = torch.empty(nb, dtype=torch.float64, device="cuda")
    assert B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 0, nb, u, nb, None, it, rel, check_conv=True) == 0
    assert rel.max().item() <= 1e-12 and torch.isfinite(u).all()
    # multigrid-preconditioned CG with the per-level smoother weights: 13 iterations
    # on configs 2, 3, 5 and 13-14 on config 4; a regression of the cycle shows up here first
    assert it.max().item() <= 14 and it.float().mean().item() <= 13.2
    rng = np.random.default_rng(100 + cfgid)
    pick = np.sort(rng.choice(nb, size=64, replace=False))
    Y = olat.nodes(p.M, p.z, p.shift, t)[:, pick]
    ref = oracle_solves(pool, cfg, Y)
    got = u[:, torch.as_tensor(pick, device="cuda")].cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max()
    b0, h = 1234, 777
    v = torch.empty((G, h), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, b0, h, v, h)
    assert torch.equal(v, u[:, b0:b0 + h])


def _values_from_spectra(sp, bins, M):
    """v_l(j, g) = F^[g][l][b]/M of the GPU's half spectra (conjugate mirror above M/2, Z17/Z18):
    the oracle's view of a round computed from the GPU's transform.  sp [G][L][Mh][2] numpy."""
    G, L = sp.shape[:2]
    F = sp[..., 0] + 1j * sp[..., 1]
    V = np.empty((L, G, bins.shape[1]), dtype=np.complex128)
    Mh = M // 2 + 1
    for l in range(L):
        b = bins[l]
        lo = b < Mh
        V[l][:, lo] = F[:, l, b[lo]]
        V[l][:, ~lo] = np.conj(F[:, l, M - b[~lo]])
    return V / M


@pytest.mark.parametrize("cfgid,t", [(2, 5), (3, 5), (4, 2), (5, 5)])
def test_bench_round_stage_parity(B, cfgid, t):
    """One bench round on the full mesh (config 4 at t = 2, |J| = 16641: its t = 3 round has
    8e9 keys, too many for the oracle): the oracle's direct DFT of the GPU's samples at 64
    sampled nodes equals the GPU spectra (<= 1e-12); the oracle's keys, threshold, selection,
    union and resolve on the GPU spectra of all nodes equal the GPU's (keys <= 1e-12 relative
    in sqrt, decisions per Z25 with the strict set check, l* exact, values <= 1e-12)."""
    from paper_2109_04131_b200.driver import Detector
    from parity import compare_round
    cfg = config(cfgid)
    det = Detector(cfg)
    I1d = det.step1()
    I_prev, _ = det.step2(I1d, t_stop=t - 1)
    kt = I1d[t - 1]
    n_prev = I_prev.shape[0] if t > 1 else 1
    nJ = n_prev * kt.numel()
    s_t = cfg["s_local"] if t < cfg["d"] else cfg["s"]
    flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
    res = det.round(2, t, 1, I_prev.contiguous(), n_prev, kt.contiguous(), s_t, flags, want_coef=True)
    assert res.kappa_min is not None, "round must take the one-shot key path"
    M, L, G = res.plan.M, res.plan.L, det.G
    Mh = M // 2 + 1
    bins = res.bins.cpu().numpy().astype(np.int64)
    # (1) direct DFT of the GPU's own samples at 64 nodes
    rng = np.random.default_rng(7 + cfgid)
    gs = np.sort(rng.choice(G, size=min(64, G), replace=False))
    U = res.u[torch.as_tensor(gs, device="cuda")].cpu().numpy()
    sp_g = res.spectra[torch.as_tensor(gs, device="cuda")].cpu().numpy()
    ref = np.stack([odft.lattice_dft(U[:, l * M:(l + 1) * M], M, np.arange(Mh)) for l in range(L)], 1)
    got = (sp_g[..., 0] + 1j * sp_g[..., 1]) / M
    assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
    # (2) the oracle's detection stage on the GPU spectra of every node (node chunks: the values
    # of all (l, g, j) would be up to 5 GB at config 5)
    sp_all = res.spectra
    chunk = max(1, int(2e8 // (L * nJ * 16)))
    kmin = np.concatenate([odet.kappa_min(_values_from_spectra(sp_all[g0:g0 + chunk].cpu().numpy(), bins, M))
                           for g0 in range(0, G, chunk)], axis=0)
    km_g = res.kappa_min.cpu().numpy()
    assert np.abs(np.sqrt(km_g) - np.sqrt(kmin)).max() <= 1e-12 * np.sqrt(kmin.max())
    th2 = odet.theta_squared(kmin, cfg["theta_rel"], cfg.get("theta_abs", 0.0))
    D, votes = odet.select(kmin, s_t, th2)
    det_o = np.nonzero(votes > 0)[0]
    pos = -np.ones(nJ, dtype=np.int64)
    pos[det_o] = np.arange(det_o.size)
    Dr = [pos[g] for g in D]                     # resolve on the detected columns only (memory)
    V = _values_from_spectra(sp_all.cpu().numpy(), bins[:, det_o], M)
    coef_o, lstar_o = odet.resolve(V, bins[:, det_o], Dr, np.arange(det_o.size))
    ref_round = dict(D=D, det=det_o, coef=coef_o, lstar=lstar_o)
    # GPU-fed: both sides read the same spectra, so a key differs by at most the rounding of
    # x (1/M) vs x / M (<= 1 ulp of the key): a band of 1e-13 max m covers it ~1e3 times
    frag = odet.fragile(kmin, s_t, th2, band=1e-13)
    out = compare_round(res.det_g.cpu().numpy(), res.n_det_g.cpu().numpy(),
                        res.det_idx.cpu().numpy(), res.lstar.cpu().numpy(), res.coef.cpu().numpy(),
                        ref_round, frag, 1e-12 * np.abs(V).max())
    assert out["nodes_same_D"] >= out["nodes"] - int(frag.any(axis=1).sum())
    print(f"config {cfgid} t={t}: |J|={nJ} L={L} M={M} n_det={det_o.size} fragile={out['fragile']} "
          f"strict={out['strict_set_check']}")


def test_full_run_pde_config2_lockstep(B, pool):
    """Config 2 (d = 10, n = 32): the GPU's whole detection (Steps 1-2, 91 rounds, 258,687
    samples), every round checked against the oracle's own FE solves, direct DFT, keys,
    threshold, selection and union on the same candidate set (the GPU's I^(1..t-1) x I^(t)):
    plans bit-exact, every non-fragile decision equal and the round sets equal when no decision
    is fragile (Z25), final-round values <= 1e-9 of max |c| (solver tolerance).  A fragile
    decision may legitimately change a union, so the sets are carried forward from the GPU run."""
    from paper_2109_04131_b200.driver import Detector
    from parity import compare_round
    from oracle import plan as oplan
    cfg = config(2)
    stats = dict(rounds=0, strict=0, fragile=0)

    class Lockstep(Detector):
        def round(self, step, t, i, I_prev, n_prev, kt, s_tilde, flags, want_coef=False, keep_iters=False,
                  counts=True):
            res = super().round(step, t, i, I_prev, n_prev, kt, s_tilde, flags, want_coef, keep_iters)
            p = res.plan
            shift = oplan.shift(cfg["seed"], step, t, i, cfg["d"])
            assert np.array_equal(p.shift, shift)
            ktn = kt.cpu().numpy().astype(np.int64)
            if step == 1:
                J = ktn.reshape(-1, 1)
                Y = olat.nodes(p.M, [[1]], shift, 1, line_axis=t - 1)
                bins = olat.bins(J, [[1]], p.M)
            else:
                J = olat.candidates(I_prev.cpu().numpy().astype(np.int64).reshape(n_prev, t - 1), ktn)
                assert np.array_equal(p.z, oplan.z_vectors(cfg["seed"], t, i, p.M, p.L))
                Y = olat.nodes(p.M, p.z, shift, t)
                bins = olat.bins(J, p.z, p.M)
            assert np.array_equal(res.bins.cpu().numpy(), bins)
            U = oracle_solves(pool, cfg, Y)
            V = odft.round_values(U, p.M, p.L, bins)
            ref = odet.detect_round(V, bins, s_tilde, cfg["theta_rel"], want_coef=want_coef)
            frag = odet.fragile(ref["kappa_min"], s_tilde, ref["theta2"])
            cm = np.abs(ref["coef"]).max() if want_coef and ref["coef"].size else 1.0
            out = compare_round(res.det_g.cpu().numpy(), res.n_det_g.cpu().numpy(),
                                res.det_idx.cpu().numpy(),
                                res.lstar.cpu().numpy() if want_coef and res.lstar is not None else None,
                                res.coef.cpu().numpy() if want_coef and res.coef is not None else None,
                                ref, frag, 1e-9 * cm)
            stats["rounds"] += 1
            stats["strict"] += int(out["strict_set_check"])
            stats["fragile"] += out["fragile"]
            return res

    det = Lockstep(cfg)
    log = []
    I, C = det.run(log)
    assert stats["rounds"] == 91 and det.n_samples == 258687
    print(f"config 2 lockstep: {stats}")
    assert stats["strict"] >= 40                 # measured: 47 of the 91 rounds have no fragile decision
