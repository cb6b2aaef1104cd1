"""GPU: the streamed (chunked) selection of large candidate sets (usfft_lattice_keys +
usfft_detect_carry, DESIGN.md §3 Z29) gives exactly the one-shot selection: the same D_g (ties
broken by candidate index), votes and theta^2, on tie-heavy synthetic keys, on the keys of a real
lattice round, and through the whole detection on the PDE black box."""
import numpy as np
import pytest
import torch

from oracle import detect as odet

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


def _streamed(B, ctx, keys, s, chunk, theta_rel, theta_abs, kmax):
    """The driver's chunk loop on given keys [G][nJ] (the chunk keys are copied in by torch here
    instead of being produced by usfft_lattice_keys)."""
    G, nJ = keys.shape
    W = s + chunk
    merged = torch.zeros((G, W), dtype=torch.float64, device="cuda")
    carry_k = torch.zeros((G, s), dtype=torch.float64, device="cuda")
    carry_j = torch.full((G, s), -1, dtype=torch.int32, device="cuda")
    det_pos = torch.empty((G, s), dtype=torch.int32, device="cuda")
    n_det_g = torch.empty(G, dtype=torch.int32, device="cuda")
    scratch = torch.empty(W, dtype=torch.int32, device="cuda")
    for j0 in range(0, nJ, chunk):
        c = min(chunk, nJ - j0)
        merged[:, s:] = 0.0
        merged[:, s:s + c] = keys[:, j0:j0 + c]
        B.usfft_detect_select(ctx, G, W, merged, kmax, s, 0.0, 0.0, scratch, det_pos, n_det_g)
        B.usfft_detect_carry(ctx, G, s, W, merged, carry_k, carry_j, det_pos, n_det_g, j0)
    th2 = torch.empty(1, dtype=torch.float64, device="cuda")
    B.usfft_detect_select(ctx, G, s, carry_k, kmax, s, theta_rel, theta_abs, scratch, det_pos, n_det_g, th2)
    votes = torch.zeros(nJ, dtype=torch.int32, device="cuda")
    det_g = torch.empty((G, s), dtype=torch.int32, device="cuda")
    B.usfft_detect_carry(ctx, G, s, s, carry_k, None, carry_j, det_pos, n_det_g, 0, det_g, votes)
    return votes, det_g, n_det_g, th2


@pytest.mark.parametrize("G,nJ,s,chunk,levels", [(7, 1000, 20, 64, 4), (33, 5000, 100, 1000, 7),
                                                 (5, 300, 50, 256, 2), (3, 97, 120, 40, 3)])
def test_streamed_equals_one_shot_on_ties(B, ctx, G, nJ, s, chunk, levels):
    """Keys drawn from a few levels (heavy ties at the s~-th rank, zeros included): the streamed
    selection reproduces the one-shot selection and the oracle's (kappa desc, j asc) top-s~."""
    rng = np.random.default_rng(G * nJ + s)
    K = rng.integers(0, levels, size=(G, nJ)).astype(np.float64) * 0.25
    keys = torch.as_tensor(K, device="cuda")
    kmax = torch.tensor([K.max()], dtype=torch.float64, device="cuda")
    for theta_rel, theta_abs in ((0.0, 0.0), (0.7, 0.0), (0.0, 0.3)):
        v1 = torch.empty(nJ, dtype=torch.int32, device="cuda")
        d1 = torch.empty((G, s), dtype=torch.int32, device="cuda")
        n1 = torch.empty(G, dtype=torch.int32, device="cuda")
        t1 = torch.empty(1, dtype=torch.float64, device="cuda")
        B.usfft_detect_select(ctx, G, nJ, keys, kmax, s, theta_rel, theta_abs, v1, d1, n1, t1)
        v2, d2, n2, t2 = _streamed(B, ctx, keys, s, chunk, theta_rel, theta_abs, kmax)
        assert torch.equal(v1, v2) and torch.equal(d1, d2) and torch.equal(n1, n2) and torch.equal(t1, t2)
        th2 = odet.theta_squared(K, theta_rel, theta_abs)
        assert float(t1.item()) == th2
        D, votes = odet.select(K, s, th2)
        assert v2.cpu().numpy().tolist() == votes.tolist()
        for g in range(G):
            assert d2[g, :int(n2[g])].cpu().numpy().tolist() == D[g].tolist()


def test_streamed_round_matches_one_shot(B):
    """A real Step-2 round of config 1 (PDE): keys produced chunk-wise by usfft_lattice_keys, then
    the carry; det_g, n_det_g, theta^2, votes and the resolved coefficients are identical."""
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config
    out = []
    for chunk in (None, 37, 256):
        cfg = config(1)
        if chunk:
            cfg["key_chunk"] = chunk
        det = Detector(cfg)
        I1d = det.step1()
        I, coef = det.step2(I1d)
        lr = det.last_round
        out.append((I.cpu(), coef.cpu(), lr.det_g.cpu(), lr.n_det_g.cpu(), lr.theta2.cpu(), lr.votes.cpu()))
    for o in out[1:]:
        for a, b in zip(out[0], o):
            assert torch.equal(a, b)


def test_example_lognormal_large_union_streams(B):
    """The lognormal example detects every 1-D frequency and unions to |J| ~ 1e5-1e7
    candidates by t = 4 (tools/round_sizes.py); with a small key budget the rounds stream and the
    sets equal the one-shot run's up to t = 3."""
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config
    sets = []
    for kb in (None, 64 << 20):
        det = Detector(config("lognormal_example", n=16, N=8))
        if kb:
            det.KEY_BYTES = kb
        I1d = det.step1()
        I, _ = det.step2(I1d, t_stop=3)
        sets.append(I.cpu())
    assert torch.equal(sets[0], sets[1])


@pytest.mark.parametrize("G,nJ,s", [(9, 1, 1), (7, 200, 20), (13, 256, 300), (5, 513, 100), (6, 1000, 100),
                                    (3, 2048, 2047), (4, 2049, 50), (3, 5000, 300), (2, 9000, 9001)])
def test_select_vs_oracle(B, ctx, G, nJ, s):
    """Per-node selection on tie-heavy keys with zeros, s~ below, at and above |J|, through both
    kernels (one warp per node for |J| <= 2048, the CTA radix select above): D_g, votes and
    theta^2 equal the oracle's lexsort selection (Z6, Z7) exactly."""
    rng = np.random.default_rng(G * nJ + s)
    K = rng.integers(0, 5, size=(G, nJ)).astype(np.float64) * 0.125
    keys = torch.as_tensor(K, device="cuda")
    kmax = torch.tensor([max(K.max(), 1e-300)], dtype=torch.float64, device="cuda")
    for theta_rel, theta_abs in ((0.0, 0.0), (0.6, 0.0), (0.0, 0.3)):
        v = torch.empty(nJ, dtype=torch.int32, device="cuda")
        d = torch.empty((G, s), dtype=torch.int32, device="cuda")
        n = torch.empty(G, dtype=torch.int32, device="cuda")
        t = torch.empty(1, dtype=torch.float64, device="cuda")
        B.usfft_detect_select(ctx, G, nJ, keys, kmax, s, theta_rel, theta_abs, v, d, n, t)
        th2 = odet.theta_squared(K, theta_rel, theta_abs)
        assert t.item() == th2
        D, votes = odet.select(K, s, th2)
        assert v.cpu().numpy().tolist() == votes.tolist()
        for g in range(G):
            assert d[g, :int(n[g])].cpu().numpy().tolist() == D[g].tolist()
