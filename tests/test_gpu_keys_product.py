"""a8 keys through the product-set path (usfft_lattice_keys_product; k_kappa_tiled when the spectra
do not fit in L2, so each case sizes its node count from the device's L2): bit-identical to the
gather kernel (usfft_lattice_keys) on the same spectra, whole and in ragged chunks with the carry
prefilter, and <= 1e-12 (sqrt) of the oracle's kappa_min of its direct-DFT values on sampled
nodes (Alg. 1 Step 2c P:313-315, Z1, Z5, Z10)."""
import numpy as np
import pytest
import torch

from oracle import detect as odet
from oracle import dft as odft
from oracle import lattice as olat

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    from paper_2109_04131_b200 import binding
    return binding


@pytest.fixture(scope="module")
def ctx(B):
    return B.Context(0)


def _inputs(G, M, L, n_prev, n1, t, seed):
    rng = np.random.default_rng(seed)
    I_prev = np.unique(rng.integers(-40, 41, size=(3 * n_prev, t - 1)), axis=0)[:n_prev]
    kt = np.arange(-(n1 // 2), n1 - n1 // 2)
    J = olat.candidates(I_prev, kt)
    z = rng.integers(1, M, size=(L, t))
    bins = olat.bins(J, z, M)
    U = rng.standard_normal((G, L * M))
    return U, z, J, bins


@pytest.mark.parametrize("M,L,n_prev,n1,t", [(97, 7, 300, 13, 3), (401, 5, 1100, 17, 4), (2017, 3, 1400, 9, 3)])
def test_product_keys_bitexact_and_vs_oracle(B, ctx, M, L, n_prev, n1, t):
    from paper_2109_04131_b200.binding import Plan
    Mh = M // 2 + 1
    # enough nodes that the spectra [G][L][Mh] complex exceed 3/4 of L2: the tiled kernel runs
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    G = (3 * l2 // 4) // (16 * L * Mh) + 7
    U, z, J, bins = _inputs(G, M, L, n_prev, n1, t, seed=M)
    nJ = J.shape[0]
    assert 4 * 16 * G * L * Mh > 3 * l2
    p = Plan(t, M, L, t, -1, z, np.zeros(t))
    spectra = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    kmax0 = torch.zeros(1, dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, G, torch.as_tensor(U, device="cuda"), [0, L * M], None, 0, spectra, None, kmax0)
    bd = torch.as_tensor(bins, dtype=torch.int32, device="cuda").contiguous()
    k_g = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
    k_p = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
    m_g = torch.zeros(1, dtype=torch.float64, device="cuda")
    m_p = torch.zeros(1, dtype=torch.float64, device="cuda")
    B.usfft_lattice_keys(ctx, p, G, spectra, bd, nJ, nJ, k_g, nJ, m_g)
    B.usfft_lattice_keys_product(ctx, p, G, spectra, bd, nJ, 0, nJ, n1, k_p, nJ, m_p)
    assert torch.equal(k_p, k_g) and m_p.item() == m_g.item()
    km = k_p.cpu().numpy()
    pick = np.sort(np.random.default_rng(M).choice(G, size=4, replace=False))     # the oracle on 4 nodes
    ref = odet.kappa_min(odft.round_values(U[pick], M, L, bins))
    assert np.abs(np.sqrt(km[pick]) - np.sqrt(ref)).max() <= 1e-12 * np.sqrt(ref.max())
    # a ragged chunk at an offset, written behind a carry of width s (the streamed layout, Z29),
    # with the carry prefilter tau
    s, j0 = 11, nJ // 3 + 5
    c = min(4 * Mh + 123, nJ - j0)
    W = s + c
    tau = torch.as_tensor(np.quantile(km[:, j0:j0 + c], 0.5, axis=1), device="cuda").contiguous()
    out_g = torch.full((G, W), -1.0, dtype=torch.float64, device="cuda")
    out_p = torch.full((G, W), -1.0, dtype=torch.float64, device="cuda")
    B.usfft_lattice_keys(ctx, p, G, spectra, bd, nJ, c, out_g, W, m_g, bins_off=j0, kmin_off=s, tau=tau)
    B.usfft_lattice_keys_product(ctx, p, G, spectra, bd, nJ, j0, c, n1, out_p, W, m_p, kmin_off=s, tau=tau)
    assert torch.equal(out_p, out_g)
    assert bool((out_p[:, :s] == -1.0).all())


@pytest.mark.parametrize("G,nJ,s,npos", [(4, 30000, 100, 1500), (3, 20000, 50, 5000), (2, 9000, 300, 250)])
def test_select_sparse_rows_bitexact(B, ctx, G, nJ, s, npos):
    """usfft_detect_select on rows longer than the staging limit whose keys are mostly 0 (the
    streamed chunks after the carry prefilter, Z29): the compacted path (<= 2048 positive keys)
    and the full-row path both give the oracle's D_g and votes exactly (ties by index, Z6)."""
    rng = np.random.default_rng(nJ + npos)
    km = np.zeros((G, nJ))
    vals = np.r_[rng.random(40), 1e-13, 0.5, 0.5]            # repeated values: ties
    for g in range(G):
        idx = rng.choice(nJ, size=npos, replace=False)
        km[g, idx] = rng.choice(vals, size=npos)
    kmax_h = km.max()
    th2_ref = odet.theta_squared(km, 1e-6)
    D, votes_ref = odet.select(km, s, th2_ref)
    kmd = torch.as_tensor(km, device="cuda")
    votes = torch.empty(nJ, dtype=torch.int32, device="cuda")
    det_g = torch.empty((G, s), dtype=torch.int32, device="cuda")
    ndg = torch.empty(G, dtype=torch.int32, device="cuda")
    th2 = torch.empty(1, dtype=torch.float64, device="cuda")
    B.usfft_detect_select(ctx, G, nJ, kmd, torch.tensor([kmax_h], dtype=torch.float64, device="cuda"), s, 1e-6,
                          0.0, votes, det_g, ndg, th2)
    assert th2.item() == th2_ref
    assert np.array_equal(votes.cpu().numpy(), votes_ref)
    dg, nd = det_g.cpu().numpy(), ndg.cpu().numpy()
    for g in range(G):
        assert dg[g, :nd[g]].tolist() == D[g].tolist()
        assert np.all(dg[g, nd[g]:] == -1)
