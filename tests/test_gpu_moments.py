"""GPU parity of usfft_moments (expectation, variance, GSI, Z30) against
oracle/moments.py on the same inputs: random sets and coefficients for every periodization, and
the output of a whole run."""
import numpy as np
import pytest
import torch

from oracle import moments as omom

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


@pytest.mark.parametrize("theta,delta", [("sin", 0.0), ("tent", 0.0), ("phi_delta", 1.0 / 1604)])
@pytest.mark.parametrize("nI,d,G", [(1, 3, 5), (300, 10, 37), (2500, 20, 300)])
def test_moments_parity(B, ctx, theta, delta, nI, d, G):
    rng = np.random.default_rng(nI + d)
    rows = {tuple([0] * d)}
    while len(rows) < nI:
        rows.add(tuple(int(v) for v in rng.integers(-9, 10, size=d) * (rng.random(d) < 0.3)))
    I = np.array(sorted(rows), dtype=np.int64)
    C = rng.standard_normal((G, nI)) + 1j * rng.standard_normal((G, nI))
    C[0] = 0.0                                                    # sigma^2 = 0 node
    C[1, (I != 0).any(1)] = 0.0                                   # constant node
    Ct = torch.as_tensor(np.stack([C.real, C.imag], -1), device="cuda").contiguous()
    It = torch.as_tensor(I, dtype=torch.int16, device="cuda")
    E = torch.empty((G, 2), dtype=torch.float64, device="cuda")
    var = torch.empty(G, dtype=torch.float64, device="cuda")
    gsi = torch.empty((G, d), dtype=torch.float64, device="cuda")
    B.usfft_moments(ctx, It, Ct, theta, delta, E, var, gsi)
    e = E.cpu().numpy()
    eo = omom.expectation(I, C, theta, delta)
    scale = np.abs(C).sum(1).max()
    assert np.abs(e[:, 0] + 1j * e[:, 1] - eo).max() <= 1e-13 * scale
    vo = omom.variance(I, C)
    assert np.abs(var.cpu().numpy() - vo).max() <= 1e-13 * vo.max()
    assert np.abs(gsi.cpu().numpy() - omom.gsi(I, C)).max() <= 1e-13
    assert not gsi[0].any() and not gsi[1].any()


def test_moments_of_a_run(B):
    """Config 1 (periodic): E is the real part of c_0 bit for bit, sum_l rho(J_l) = 1 per node,
    and the values equal the oracle's on the run's own I and coefficients."""
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config
    cfg = config(1)
    det = Detector(cfg)
    I, coef = det.run()
    E, var, gsi = det.moments(I, coef)
    Ih = I.cpu().numpy().astype(np.int64)
    c = coef.cpu().numpy()
    C = c[..., 0] + 1j * c[..., 1]
    z = np.nonzero((Ih == 0).all(1))[0][0]
    assert torch.equal(E[:, 0].cpu(), coef[:, z, 0].cpu())
    assert np.allclose(gsi.sum(1).cpu().numpy(), 1.0, rtol=0, atol=1e-12)
    assert np.abs(var.cpu().numpy() - omom.variance(Ih, C)).max() <= 1e-13 * var.max().item()
