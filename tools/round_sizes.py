"""Print every detection round's sizes as it finishes (M, L, |J|, detected, union) for one
workload: python tools/round_sizes.py --config lognormal_example [--n 32] [--N 32] [--s 100]."""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


class _Log(list):
    def append(self, x):
        super().append(x)
        print(json.dumps(x), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--N", type=int, default=0)
    ap.add_argument("--s", type=int, default=0)
    ap.add_argument("--t-stop", type=int, default=0)
    ap.add_argument("--theta-rel", type=float, default=-1.0, help="relative threshold (switches off theta_abs)")
    ap.add_argument("--mode", default="", help="Algorithm A mode override (A or R)")
    ap.add_argument("--quiet", action="store_true", help="only the per-t union sizes")
    args = ap.parse_args()
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config
    cfg = config(int(args.config) if args.config.isdigit() else args.config)
    if args.n:
        cfg["n"] = args.n
    if args.N:
        cfg["N"] = args.N
    if args.s:
        cfg["s"] = cfg["s_local"] = args.s
    if args.mode:
        cfg["mode"] = args.mode
    if args.theta_rel >= 0:
        cfg["theta_rel"], cfg["theta_abs"] = args.theta_rel, 0.0
    det = Detector(cfg)
    det.timing = True
    orig = det.round

    def timed_round(*a, **k):
        res = orig(*a, **k)
        if not args.quiet:
            print(json.dumps({"times_ms": {k2: round(v, 3) for k2, v in res.times.items()},
                              "chunked": det.key_chunk(res.nJ, a[6]) is not None}), flush=True)
        return res
    det.round = timed_round
    log = _Log()
    I1d = det.step1(log)
    print(json.dumps({"I1d_sizes": [int(v.numel()) for v in I1d]}), flush=True)
    I, _ = det.step2(I1d, log, t_stop=args.t_stop or None)
    print(json.dumps({"nI": int(I.shape[0])}), flush=True)


if __name__ == "__main__":
    main()
