"""Checkpoint / resume of a detection run: a run interrupted after a
dimension of Step 2 and resumed from its checkpoint gives the uninterrupted run's frequency set
and coefficients bit for bit (all randomness is counter-based, Z4)."""
import numpy as np
import pytest
import torch

from usfft_inputs import config

pytestmark = pytest.mark.gpu


def test_resume_matches_uninterrupted_run(tmp_path):
    from paper_2109_04131_b200.driver import Detector
    cfg = config(1, mode="A")
    I_full, C_full = Detector(cfg).run()
    path = str(tmp_path / "cfg1.npz")
    det = Detector(cfg)
    I1d = det.step1()
    det.save_checkpoint(path, I1d, 1, None)
    det.step2(I1d, t_stop=2, checkpoint=path)           # "interrupted" after t = 2
    I1d_c, t0, I_prev = Detector(cfg).load_checkpoint(path)
    assert t0 == 2 and I_prev.shape[1] == 2
    assert all(torch.equal(a, b) for a, b in zip(I1d, I1d_c))
    I_res, C_res = Detector(cfg).run(checkpoint=path)   # resumes at t = 3
    assert torch.equal(I_res, I_full)
    assert np.array_equal(C_res.cpu().numpy(), C_full.cpu().numpy())


def test_checkpoint_of_another_config_is_refused(tmp_path):
    from paper_2109_04131_b200.driver import Detector
    cfg = config(1, mode="A")
    det = Detector(cfg)
    I1d = [torch.zeros(1, dtype=torch.int16, device="cuda")] * cfg["d"]
    path = str(tmp_path / "x.npz")
    det.save_checkpoint(path, I1d, 1, None)
    other = dict(cfg, seed=cfg["seed"] + 1)
    with pytest.raises(ValueError):
        Detector(other).load_checkpoint(path)


def test_unsynchronised_rounds_match_synchronised_rounds():
    """The rounds i < r of a Step-2 dimension are enqueued without a host synchronisation
    (usfft_detect_union with n_det == NULL); a run that synchronises after every round (log
    requested) must give the same frequency set and coefficients bit for bit."""
    from paper_2109_04131_b200.driver import Detector
    cfg = config(1, mode="A")
    log = []
    I_sync, C_sync = Detector(cfg).run(log=log)
    I_async, C_async = Detector(cfg).run()
    assert any(e["step"] == 2 and e["i"] > 1 for e in log)          # the workload has r > 1 rounds
    assert torch.equal(I_sync, I_async)
    assert np.array_equal(C_sync.cpu().numpy(), C_async.cpu().numpy())
