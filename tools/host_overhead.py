"""Host-side cost per C-ABI call (wall clock of back-to-back calls, GPU work tiny): to size the
launch overheads of the round.  python tools/host_overhead.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2109_04131_b200 import binding as B
    from usfft_inputs import config
    cfg = config(2)
    ctx = B.Context(0)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
    G = 961
    pde = B.pde_desc(cfg)
    u = torch.empty((G, 4), dtype=torch.float64, device="cuda")
    kt = torch.arange(-3, 4, dtype=torch.int16, device="cuda")
    Ip = torch.zeros((1, 4), dtype=torch.int16, device="cuda")
    bins = torch.empty((p.L, 7), dtype=torch.int32, device="cuda")
    km = torch.rand((G, 100), dtype=torch.float64, device="cuda")
    kmax = torch.ones(1, dtype=torch.float64, device="cuda")
    votes = torch.empty(100, dtype=torch.int32, device="cuda")
    dg = torch.empty((G, 20), dtype=torch.int32, device="cuda")
    nd = torch.empty(G, dtype=torch.int32, device="cuda")
    calls = {
        "plan_round": lambda: B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000),
        "sample_pde(nb=4)": lambda: B.usfft_sample_pde(ctx, pde, p, 0, 4, u, 4),
        "lattice(bins)": lambda: B.usfft_lattice(ctx, p, 0, 0, None, Ip, 1, kt, bins),
        "detect_select": lambda: B.usfft_detect_select(ctx, G, 100, km, kmax, 20, 1e-6, 0.0, votes, dg, nd),
        "torch.zeros": lambda: torch.zeros(1000, dtype=torch.uint8, device="cuda"),
    }
    for name, f in calls.items():
        for _ in range(20):
            f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(200):
            f()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{name:18s} {1e6 * (t1 - t0) / 200:8.1f} us/call (host)")


if __name__ == "__main__":
    main()
