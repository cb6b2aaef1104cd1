"""Small invocations of every hot-path kernel for compute-sanitizer (one tool per gpurun call, the
B200 profiling guide): python tools/sanitize_run.py
  smoke round of config 1 (k_pcg_mg n = 16, k_nodes/k_bins, Rader M = 97, keys, select, union,
  resolve); k_pcg_mg n = 32; k_pcg_cl n = 64 and n = 128 (clusters, DSMEM, mbarriers) on a few
  samples; the lattice FFT k_fft_rader_r at M = 401 and 4001 and k_fft_rader_tp at M = 2017."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import __graft_entry__ as ge
    from paper_2109_04131_b200 import binding as B
    from usfft_inputs import config
    ge.smoke()
    print("smoke ok", flush=True)
    ctx = B.Context(0)
    for cfgid, nb in ((2, 6), (3, 6), (5, 4)):
        cfg = config(cfgid)
        p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
        G = (cfg["n"] - 1) ** 2
        u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
        it = torch.empty(nb, dtype=torch.int32, device="cuda")
        B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 0, nb, u, nb, None, it)
        torch.cuda.synchronize()
        print(f"pde config {cfgid} ok, iterations {it.tolist()}", flush=True)
    for G, M, L in ((5, 401, 3), (3, 2017, 2), (2, 4001, 3)):
        p = B.Plan(3, M, L, 3, -1, np.ones((L, 3), dtype=np.int64), np.zeros(3))
        x = torch.randn((G, L * M), dtype=torch.float64, device="cuda")
        sp = torch.empty((G, L, M // 2 + 1, 2), dtype=torch.float64, device="cuda")
        B.usfft_lattice_fft(ctx, p, G, x, [0, L * M], None, 0, sp, None, None)
        torch.cuda.synchronize()
        print(f"fft M = {M} ok", flush=True)


if __name__ == "__main__":
    main()
