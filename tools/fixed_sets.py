"""Sec. 4.5 comparison: Step 3 + the accuracy metric on a-priori frequency sets
(axis cross, hyperbolic crosses, weighted l1-balls) instead of the detected set, for one
workload; one JSON line per (set, N).

    python tools/fixed_sets.py --config periodic_mu1.2 [--N 4 8 16 32] [--n-test 10000]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

FAMILIES = [("axis", 1), ("hc_uniform", 1), ("hc", 1), ("hc", 2), ("l1", 1), ("l1", 2)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="periodic_mu1.2")
    ap.add_argument("--N", type=int, nargs="+", default=[4, 8, 16, 32])
    ap.add_argument("--n-test", type=int, default=10000)
    ap.add_argument("--max-set", type=int, default=60000)
    args = ap.parse_args()
    import torch
    from paper_2109_04131_b200.driver import Detector
    from paper_2109_04131_b200.index_sets import frequency_set
    from usfft_inputs import config, uniform_points

    key = int(args.config) if args.config.isdigit() else args.config
    cfg = config(key)
    d = cfg["d"]
    Y = torch.as_tensor(uniform_points(2000 + cfg["seed"], d, args.n_test), dtype=torch.float64, device="cuda")
    U_check = None
    for kind, q in FAMILIES:
        for N in args.N:
            try:
                I = frequency_set(kind, d, N, q, limit=args.max_set)
            except ValueError:
                print(json.dumps({"set": kind, "q": q, "N": N, "skipped": f"more than {args.max_set} frequencies"}))
                continue
            det = Detector(dict(cfg, N=max(N, 1)))
            t0 = time.perf_counter()
            It = torch.as_tensor(I, dtype=torch.int16, device="cuda")
            cov, coef = det.step3(It)
            err, U = det.errors(It, coef, Y) if U_check is None else (None, U_check)
            if err is None:
                err = torch.empty((coef.shape[0], 3), dtype=torch.float64, device="cuda")
                from paper_2109_04131_b200 import binding as B
                B.usfft_eval_err(det.ctx, It, coef, Y, U_check, err)
            U_check = U
            torch.cuda.synchronize()
            e = err.cpu().numpy()
            print(json.dumps({"workload": cfg["name"], "set": kind, "q": q, "N": N, "nI": int(I.shape[0]),
                              "samples": int(det.n_samples), "cover_lattices": int(cov.z.shape[0]),
                              "err2_max": float(e[:, 1].max()), "errinf_max": float(e[:, 2].max()),
                              "wall_s": time.perf_counter() - t0}), flush=True)


if __name__ == "__main__":
    main()
