"""Whole Alg. 1 on one workload: Steps 1-2 (detection), Step 3 (multiple-R1L coefficients) and
the accuracy metric err_1 / err_2 / err_inf at n_test uniform test parameters.

    python tools/full_run.py [--config 2] [--n-test 10000]

Prints one JSON line: samples per step, times (CUDA events), |I| and q = |I| / s (Remark on
P:1613-1619), and the errors (max and mean over the nodes chi_g).  Single GPU.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2", help="BASELINE config 1-5 or an example preset name")
    ap.add_argument("--n-test", type=int, default=10000)
    ap.add_argument("--theta", default="", help="coefficient map override (sin, tent, probit, phi_delta)")
    ap.add_argument("--form", default="", help="coefficient form override (affine, exp)")
    ap.add_argument("--lattice-factor", type=int, default=1, help="Step-2 lattices sized for f s~ (Z2 x f)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config, uniform_points

    key = int(args.config) if args.config.isdigit() else args.config
    cfg = config(key)
    if args.theta:
        cfg["theta"] = args.theta
    if args.form:
        cfg["form"] = args.form
    if args.lattice_factor > 1:
        cfg["lattice_factor"] = args.lattice_factor
    det = Detector(cfg)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t0 = time.perf_counter()
    ev[0].record()
    log = []
    I, _ = det.run(log)
    ev[1].record()
    n_detect = det.n_samples
    cov, coef = det.step3(I)
    ev[2].record()
    n_step3 = det.n_samples - n_detect
    Y = torch.as_tensor(uniform_points(1000 + (key if isinstance(key, int) else cfg["seed"]), cfg["d"], args.n_test), dtype=torch.float64,
                        device="cuda")
    err, _ = det.errors(I, coef, Y)
    ev[3].record()
    Em, var, gsi = det.moments(I, coef) if cfg["theta"] in ("sin", "tent", "phi_delta") else (None, None, None)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    e = err.cpu().numpy()
    out = {
        "workload": (f"config{key}" if isinstance(key, int) else "example") + f":{cfg['name']}", "theta": cfg["theta"], "form": cfg["form"],
        "delta": det.delta, "lattice_factor": args.lattice_factor, "d": cfg["d"], "n": cfg["n"], "N": cfg["N"],
        "s": cfg["s"], "rounds": len(log), "samples_detection": n_detect, "samples_step3": n_step3,
        "step3_share": n_step3 / (n_detect + n_step3), "nI": int(I.shape[0]), "q": I.shape[0] / cfg["s"],
        "cover_lattices": int(cov.z.shape[0]), "cover_M": int(cov.M),
        "ms_detection": ev[0].elapsed_time(ev[1]), "ms_step3": ev[1].elapsed_time(ev[2]),
        "ms_errors": ev[2].elapsed_time(ev[3]), "wall_s": wall, "n_test": args.n_test,
        "err1_max": float(e[:, 0].max()), "err2_max": float(e[:, 1].max()), "errinf_max": float(e[:, 2].max()),
        "err2_mean": float(e[:, 1].mean()),
    }
    if gsi is not None:                                  # post-processing (Z30)
        gh = gsi.cpu().numpy()
        Ih = I.cpu().numpy()
        nnz = (Ih != 0).sum(1)
        out.update({"J_l_sizes": [int((nnz == l).sum()) for l in range(1, 5)],
                    "gsi_J1_min": float(gh[:, 0].min()), "gsi_J1_median": float(np.median(gh[:, 0])),
                    "gsi_mean_l1_4": [float(v) for v in gh[:, :4].mean(0)],
                    "E_max": float(Em[:, 0].max()), "E_imag_max": float(Em[:, 1].abs().max())})
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
