"""Experiment: per-round detections of one Step-2 round (t = 2) under alternative detection keys
computed from the round's spectra (torch, not the product path): min over lattices (Z1, the
product), lower median, mean; vs mode R.  python tools/key_study.py --config lognormal_example"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="lognormal_example")
    ap.add_argument("--t", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config
    cfg = config(int(args.config) if args.config.isdigit() else args.config)
    det = Detector(cfg)
    I1d = det.step1()
    I_prev, _ = det.step2(I1d, t_stop=args.t - 1) if args.t > 2 else (I1d[0].reshape(-1, 1).contiguous(), None)
    kt = I1d[args.t - 1]
    n_prev = I_prev.shape[0]
    nJ = n_prev * kt.numel()
    s = cfg["s_local"]
    out = {"nJ": nJ}
    unions = {}
    for i in range(1, cfg["r"] + 1):
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        res = det.round(2, args.t, i, I_prev, n_prev, kt, s, flags)
        M, L = res.plan.M, res.plan.L
        Mh = M // 2 + 1
        sp = res.spectra                                  # [G][L][Mh][2]
        b = res.bins.long()                               # [L][nJ]
        fold = torch.where(b < Mh, b, M - b)
        G = sp.shape[0]
        vals = torch.stack([sp[:, l, fold[l], :] for l in range(L)], 1) / M     # [G][L][nJ][2]
        mag2 = (vals ** 2).sum(-1)                        # [G][L][nJ]
        keys = {"min": mag2.min(1).values, "median": mag2.median(1).values, "mean": mag2.mean(1)}
        for name, k in keys.items():
            top = torch.topk(k, s, dim=1).indices          # per node top-s
            sel = torch.zeros(nJ, dtype=torch.bool, device="cuda")
            sel[top.reshape(-1)] = True
            unions.setdefault(name, torch.zeros(nJ, dtype=torch.bool, device="cuda"))
            unions[name] |= sel
            out[f"{name}_round{i}"] = int(sel.sum())
        out[f"product_round{i}"] = res.n_det
    for name, u in unions.items():
        out[f"{name}_union"] = int(u.sum())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
