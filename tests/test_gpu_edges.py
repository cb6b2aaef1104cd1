"""GPU edge cases of the C-ABI: empty and ragged inputs, non-prime / tiny lattice sizes (direct DFT
path), argument errors (EINVAL, nothing written), determinism of repeated calls."""
import numpy as np
import pytest
import torch

from oracle import dft as odft
from oracle import lattice as olat

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


def test_empty_ranges(B, ctx):
    from usfft_inputs import config
    cfg = config(1)
    p = B.usfft_plan_round(ctx, 0, 2, 2, 1, 4, 8, 20, "A", 30)
    u = torch.zeros((225, 1), dtype=torch.float64, device="cuda")
    assert B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 5, 0, u, 1, check_conv=True) == 0
    km = torch.zeros(1, dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, 0, u, [0, p.L * p.M], None, 0, None, None, km)
    assert km.item() == 0.0
    n_det, n_u = B.usfft_detect_union(ctx, 0, None, None, None)
    assert (n_det, n_u) == (0, 0)


@pytest.mark.parametrize("M", [2, 3, 17, 65, 129, 97])
def test_small_and_composite_lattice_sizes(B, ctx, M):
    """Step-1 line lattices have M = K = 2N+1 (composite: direct DFT kernel; prime: Rader)."""
    from paper_2109_04131_b200.binding import Plan
    rng = np.random.default_rng(M)
    G, L = 3, 1
    U = rng.standard_normal((G, M))
    J = np.arange(-(M // 2), M - M // 2).reshape(-1, 1)
    bins = olat.bins(J, [[1]], M)
    p = Plan(1, M, L, 1, 0, np.array([[1]]), np.zeros(1))
    Mh = M // 2 + 1
    sp = torch.empty((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    km = torch.empty((G, J.shape[0]), dtype=torch.float64, device="cuda")
    kx = torch.empty(1, dtype=torch.float64, device="cuda")
    B.usfft_lattice_fft(ctx, p, G, dev(U, torch.float64), [0, M], dev(bins, torch.int32), J.shape[0], sp, km, kx)
    ref = odft.lattice_dft(U, M, np.arange(Mh)) * M
    got = sp.cpu().numpy()[:, 0]
    assert np.abs(got[..., 0] + 1j * got[..., 1] - ref).max() <= 1e-12 * np.abs(ref).max()


def test_invalid_arguments_raise_einval(B, ctx):
    from paper_2109_04131_b200.binding import Plan, UsfftError
    bad = Plan(2, 5, 1, 2, -1, np.array([[7, 1]]), np.zeros(2))          # z outside [0, M)
    nodes = torch.full((2, 5), -1.0, dtype=torch.float64, device="cuda")
    with pytest.raises(UsfftError) as e:
        B.usfft_lattice(ctx, bad, 0, 5, nodes)
    assert e.value.status == 1
    assert torch.all(nodes == -1.0)                                      # nothing written
    bad_shift = Plan(2, 5, 1, 2, -1, np.array([[1, 2]]), np.array([0.5, 1.5]))
    with pytest.raises(UsfftError):
        B.usfft_lattice(ctx, bad_shift, 0, 5, nodes)
    ok = Plan(2, 5, 1, 2, -1, np.array([[1, 2]]), np.zeros(2))
    with pytest.raises(UsfftError):                                      # sample range beyond L*M
        B.usfft_lattice(ctx, ok, 3, 5, nodes)
    assert torch.all(nodes == -1.0)
    # the ctx stays usable after EINVAL (not sticky)
    B.usfft_lattice(ctx, ok, 0, 5, nodes)
    assert np.array_equal(nodes.cpu().numpy(), olat.nodes(5, [[1, 2]], [0.0, 0.0], 2))


def test_repeated_calls_bit_identical(B, ctx):
    from usfft_inputs import config
    cfg = config(2)
    p = B.usfft_plan_round(ctx, 1, 2, 3, 1, 10, 32, 100, "A", 500)
    out = []
    for _ in range(2):
        u = torch.empty((961, 40), dtype=torch.float64, device="cuda")
        B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 7, 40, u, 40)
        out.append(u)
    assert torch.equal(out[0], out[1])


def test_gather_rows_step1(B, ctx):
    kt = dev(np.arange(-5, 6), torch.int16)
    idx = dev(np.array([0, 3, 10]), torch.int32)
    rows = torch.empty((3, 1), dtype=torch.int16, device="cuda")
    B.usfft_gather_rows(ctx, idx, 3, None, 1, kt, rows)
    assert rows.reshape(-1).tolist() == [-5, -2, 5]
    Ip = dev(np.array([[1, 2], [3, 4]]), torch.int16)
    kt2 = dev(np.array([7, 8, 9]), torch.int16)
    idx2 = dev(np.array([1, 5]), torch.int32)
    rows2 = torch.empty((2, 3), dtype=torch.int16, device="cuda")
    B.usfft_gather_rows(ctx, idx2, 2, Ip, 3, kt2, rows2)
    assert rows2.tolist() == [[1, 2, 8], [3, 4, 9]]


def test_new_entry_points_validate(B, ctx):
    """EINVAL / EUNIMPL paths of the round's later entry points (nothing launched, ctx usable)."""
    from paper_2109_04131_b200.binding import UsfftError
    from usfft_inputs import config
    I = torch.zeros((2, 3), dtype=torch.int16, device="cuda")
    C = torch.zeros((4, 2, 2), dtype=torch.float64, device="cuda")
    E = torch.full((4, 2), 7.0, dtype=torch.float64, device="cuda")
    var = torch.empty(4, dtype=torch.float64, device="cuda")
    with pytest.raises(UsfftError):                                   # clipped Phi^-1: no D_k
        B.usfft_moments(ctx, I, C, "probit", 0.0, E, var)
    assert torch.all(E == 7.0)
    with pytest.raises(UsfftError):                                   # phi_Delta needs Delta
        B.usfft_moments(ctx, I, C, "phi_delta", 0.0, E, var)
    B.usfft_moments(ctx, I, C, "tent", 0.0, E, var)                  # C = 0 -> E = 0, var = 0
    assert not E.any() and not var.any()
    cfg = config(1, n=20)
    p = B.usfft_plan_round(ctx, 0, 2, 2, 1, 4, 8, 20, "A", 30)
    u = torch.empty((19 * 19, 2), dtype=torch.float64, device="cuda")
    with pytest.raises(UsfftError) as e:                              # multigrid needs a power of two
        B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond="mg"), p, 0, 2, u, 2)
    assert e.value.status != 0
    bad = B.pde_desc(config(1))
    bad[0].psi = 7
    with pytest.raises(UsfftError):
        B.usfft_sample_pde(ctx, bad, p, 0, 2, torch.empty((225, 2), dtype=torch.float64, device="cuda"), 2)
    km = torch.empty((3, 10), dtype=torch.float64, device="cuda")
    sp = torch.zeros((3, p.L, p.M // 2 + 1, 2), dtype=torch.float64, device="cuda")
    bins = torch.zeros((p.L, 10), dtype=torch.int32, device="cuda")
    kx = torch.zeros(1, dtype=torch.float64, device="cuda")
    with pytest.raises(UsfftError):                                   # ldk < nJ
        B.usfft_lattice_keys(ctx, p, 3, sp, bins, 10, 10, km, 5, kx)
    B.usfft_lattice_keys(ctx, p, 3, sp, bins, 10, 10, km, 10, kx)    # zero spectra -> zero keys
    assert not km.any()
    dp = torch.zeros((3, 4), dtype=torch.int32, device="cuda")
    nd = torch.zeros(3, dtype=torch.int32, device="cuda")
    cj = torch.full((3, 4), -1, dtype=torch.int32, device="cuda")
    with pytest.raises(UsfftError):                                   # width < s~
        B.usfft_detect_carry(ctx, 3, 4, 3, km, km, cj, dp, nd, 0)


def test_maximum_parameter_dimension(B, ctx):
    """d = 64 (kMaxD) coefficient terms on n = 16: samples match the oracle (the psi tables and
    th_amp at their largest)."""
    from oracle import fe as ofe
    cfg = dict(n=16, d=64, amp=[0.3 / (j * j) for j in range(1, 65)], theta="sin", form="affine", f="x2")
    p = B.usfft_plan_round(ctx, 3, 2, 2, 1, 64, 4, 10, "A", 30)
    nb = 5
    u = torch.empty((225, nb), dtype=torch.float64, device="cuda")
    for precond in ("mg", "jacobi"):
        assert B.usfft_sample_pde(ctx, B.pde_desc(cfg, precond=precond), p, 0, nb, u, nb, check_conv=True) == 0
        ref = ofe.sample_pde(cfg, olat.nodes(p.M, p.z, p.shift, 2)[:, :nb])
        assert np.abs(u.cpu().numpy() - ref).max() <= 1e-10 * np.abs(ref).max()


def test_union_without_counts(B, ctx):
    """usfft_detect_union with n_det == NULL: no host outputs, same device outputs as the
    synchronising call; n_union without n_det is refused (include/usfft.h, a11)."""
    import ctypes as C
    rng = np.random.default_rng(5)
    nJ = 5000
    votes_h = (rng.random(nJ) < 0.1).astype(np.int32) * rng.integers(1, 9, nJ).astype(np.int32)
    outs = []
    for counts in (True, False):
        votes = dev(votes_h, torch.int32)
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        flags[::7] = 1                                       # a running union from earlier rounds
        det_idx = torch.full((nJ,), -1, dtype=torch.int32, device="cuda")
        union_idx = torch.full((nJ,), -1, dtype=torch.int32, device="cuda")
        nd, nu = B.usfft_detect_union(ctx, nJ, votes, flags, det_idx, union_idx, counts=counts)
        torch.cuda.synchronize()
        outs.append((nd, nu, flags.cpu().numpy(), det_idx.cpu().numpy(), union_idx.cpu().numpy()))
    (nd, nu, f0, d0, u0), (nd1, nu1, f1, d1, u1) = outs
    assert (nd1, nu1) == (None, None)
    expect = (votes_h > 0) | (np.arange(nJ) % 7 == 0)
    assert nd == int((votes_h > 0).sum()) and nu == int(expect.sum())
    assert np.array_equal(f0, expect.astype(np.uint8)) and np.array_equal(f1, f0)
    assert np.array_equal(d1[:nd], d0[:nd]) and np.array_equal(u1[:nu], u0[:nu])
    assert np.array_equal(d0[:nd], np.flatnonzero(votes_h > 0)) and np.array_equal(u0[:nu], np.flatnonzero(expect))
    votes = dev(votes_h, torch.int32)
    flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
    nu_c = C.c_int64(0)
    st = ctx.lib.usfft_detect_union(ctx.h, nJ, votes.data_ptr(), flags.data_ptr(), det_idx.data_ptr(), None,
                                    union_idx.data_ptr(), C.byref(nu_c))
    assert st != 0 and "n_union without n_det" in ctx.last_error()
