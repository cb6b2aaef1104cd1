"""Two and three ranks on one GPU: the whole multi-rank driver path — sample sharding, the
transpose into node slabs, kappa_max MAX, votes SUM, per-rank resolve, Step 3, the accuracy
metric and the moments — gives the single-process result bit for bit (all
exchanges are data movement or order-free).
  * loopback: the library's own data plane (usfft_transpose and the collectives inside
    usfft_detect_select / usfft_detect_union) with P virtual ranks, one host thread and stream
    each, in one process (NCCL itself needs one GPU per rank);
  * gloo: P processes sharing cuda:0 with the exchanges through torch.distributed (TorchExchange).
"""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(cfg, loopback=None):
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import uniform_points
    det = Detector(cfg, loopback=loopback)
    I, coef = det.run()
    cov, c3 = det.step3(I)
    Y = torch.as_tensor(uniform_points(17, cfg["d"], 257), dtype=torch.float64, device="cuda")
    err, _ = det.errors(I, c3, Y)                               # test solves sharded over ranks
    E, var, gsi = det.moments(I, c3)
    return (I.cpu().numpy(), coef.cpu().numpy(), c3.cpu().numpy(), err.cpu().numpy(),
            torch.cat([E, var[:, None], gsi], 1).cpu().numpy(), det.g0, det.g1)


def _worker(rank, world, port, cfg, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        q.put((rank, _run(cfg)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,key_chunk", [(2, 0), (3, 0), (2, 64)])
def test_multirank_detector_matches_single_process(world, key_chunk):
    """key_chunk > 0: every Step-2 selection streamed over candidate chunks (Z29) on every rank."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import torch.multiprocessing as mp
    from usfft_inputs import config
    cfg = config(1)
    if key_chunk:
        cfg["key_chunk"] = key_chunk
    ref_I, ref_coef, ref_c3, ref_err, ref_mom, _, _ = _run(cfg)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(world):
        I, coef, c3, err, mom, g0, g1 = res[r]
        assert np.array_equal(I, ref_I)                       # identical detected set on every rank
        assert np.array_equal(coef, ref_coef[g0:g1])          # this rank's nodes, bit for bit
        assert np.array_equal(c3, ref_c3[g0:g1])
        assert np.array_equal(err, ref_err[g0:g1])            # accuracy metric of this rank's nodes
        assert np.array_equal(mom, ref_mom[g0:g1])            # expectation, variance, GSI


@pytest.mark.parametrize("world,key_chunk", [(2, 0), (3, 0), (3, 64)])
def test_loopback_library_collectives_match_single_process(world, key_chunk):
    """P virtual ranks in threads on one GPU, every exchange inside libusfft (loopback hub):
    identical detected set on every rank and every rank's coefficients, Step-3 coefficients,
    errors and moments equal the single-process rows bit for bit."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import threading
    from usfft_inputs import config
    cfg = config(1)
    if key_chunk:
        cfg["key_chunk"] = key_chunk
    ref_I, ref_coef, ref_c3, ref_err, ref_mom, _, _ = _run(cfg)
    key = os.urandom(128)
    res, errs = {}, []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                res[r] = _run(cfg, loopback=(r, world, key))
                s.synchronize()
        except Exception as e:                              # surfaced below
            errs.append(e)

    threads = [threading.Thread(target=worker, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=600)
        assert not t.is_alive(), "loopback rank hung"
    assert not errs, errs
    for r in range(world):
        I, coef, c3, err, mom, g0, g1 = res[r]
        assert np.array_equal(I, ref_I)
        assert np.array_equal(coef, ref_coef[g0:g1])
        assert np.array_equal(c3, ref_c3[g0:g1])
        assert np.array_equal(err, ref_err[g0:g1])
        assert np.array_equal(mom, ref_mom[g0:g1])
