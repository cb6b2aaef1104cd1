"""Cluster PCG (k_pcg_cl) check on the GPU: full-size batch (many samples per cluster), a random
subset against the oracle's banded Cholesky, timing.  python tools/cl_check.py --config 5"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--nb", type=int, default=0)
    ap.add_argument("--check", type=int, default=6)
    ap.add_argument("--reps", type=int, default=2)
    args = ap.parse_args()
    import torch
    from paper_2109_04131_b200 import binding as B
    from usfft_inputs import config
    from oracle import fe as ofe, lattice as olat
    cfg = config(args.config)
    ctx = B.Context(0)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
    nb = args.nb or p.L * p.M
    G = (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    it = torch.empty(nb, dtype=torch.int32, device="cuda")
    rel = torch.empty(nb, dtype=torch.float64, device="cuda")
    pde = B.pde_desc(cfg)
    t0 = time.time()
    nc = B.usfft_sample_pde(ctx, pde, p, 0, nb, u, nb, None, it, rel, check_conv=True)
    torch.cuda.synchronize()
    first = time.time() - t0
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(ctx.stream)
        B.usfft_sample_pde(ctx, pde, p, 0, nb, u, nb, None, it, rel)
        e1.record(ctx.stream)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    rng = np.random.default_rng(1)
    pick = np.sort(rng.choice(nb, size=min(args.check, nb), replace=False))
    Y = olat.nodes(p.M, p.z, p.shift, 5)[:, pick]
    t1 = time.time()
    ref = ofe.sample_pde(cfg, Y)
    t_or = time.time() - t1
    got = u.cpu().numpy()[:, pick]
    err = float(np.abs(got - ref).max() / np.abs(ref).max())
    print(json.dumps({"config": args.config, "n": cfg["n"], "nb": nb, "noconv": nc, "first_call_s": first,
                      "ms": min(ts), "samples_per_s": nb / min(ts) * 1e3, "iters_mean": float(it.float().mean()),
                      "iters_max": int(it.max()), "relres_max": float(rel.max()), "checked": pick.tolist(),
                      "max_rel_err_vs_oracle": err, "oracle_s": t_or}), flush=True)
    assert nc == 0 and err <= 1e-10


if __name__ == "__main__":
    main()
