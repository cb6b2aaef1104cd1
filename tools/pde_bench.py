"""Time usfft_sample_pde alone on one Step-2 lattice plan of a workload (CUDA events, after
warm-up): python tools/pde_bench.py --config 3 [--nb 8192] [--precond mg] [--reps 3]"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3")
    ap.add_argument("--nb", type=int, default=8192)
    ap.add_argument("--precond", default="")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--maxit", type=int, default=20000, help="cap (1: setup + one iteration)")
    args = ap.parse_args()
    import torch
    from paper_2109_04131_b200 import binding as B
    from usfft_inputs import config
    cfg = config(int(args.config) if args.config.isdigit() else args.config)
    ctx = B.Context(0)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
    nb = min(args.nb, p.L * p.M)
    G = (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    it = torch.empty(nb, dtype=torch.int32, device="cuda")
    pde = B.pde_desc(cfg, precond=args.precond or None, maxit=args.maxit)
    B.usfft_sample_pde(ctx, pde, p, 0, nb, u, nb, None, it)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        B.usfft_sample_pde(ctx, pde, p, 0, nb, u, nb, None, it)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(json.dumps({"config": args.config, "n": cfg["n"], "nb": nb, "precond": B.effective_precond(cfg, args.precond or None),
                      "ms": ms, "us_per_sample": 1e3 * ms / nb, "samples_per_s": nb / ms * 1e3,
                      "iters_mean": float(it.float().mean())}))


if __name__ == "__main__":
    main()
