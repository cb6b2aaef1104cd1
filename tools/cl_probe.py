"""Phase latencies of k_pcg_cl from a probe build (-DUSFFT_CL_PROBE): clock64() of thread 0 of
each CTA of cluster 0 at every phase boundary of CG iteration 6 and of the first sample's setup.
python tools/cl_probe.py --config 5"""
from __future__ import annotations

import argparse
import ctypes as C
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

NAMES = {0: "iteration start", 1: "X1 wait", 2: "fine residual", 3: "R1, Z1 + X2", 4: "level-1 residual",
         5: "R2 + X3", 6: "replicated down", 7: "K map", 8: "replicated up", 9: "S1",
         10: "fine post-smooth", 11: "u + X4", 12: "A u, dots + X5", 13: "update + X1 send",
         20: "setup start", 29: "theta, amp", 30: "coef table", 21: "barrier A", 22: "couplings + coarse push", 24: "replicated couplings",
         26: "K-level couplings, DK, DIK", 27: "GJ + B", 28: "C", 25: "join", 31: "BtC + 5-point", 23: "barrier C"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--nb", type=int, default=4096)
    args = ap.parse_args()
    from paper_2109_04131_b200 import _native, build
    out = "/tmp/libusfft_probe.so"
    cmd = [build.NVCC, *build.FLAGS, "-DUSFFT_CL_PROBE", "-o", out, *build.sources()]
    subprocess.run(cmd, cwd=build.SRC, check=True)
    _native.LIB_PATH = out
    import torch
    from paper_2109_04131_b200 import binding as B
    from usfft_inputs import config
    cfg = config(args.config)
    ctx = B.Context(0)
    p = B.usfft_plan_round(ctx, cfg["seed"], 2, 5, 1, cfg["d"], cfg["N"], cfg["s"], "A", 1000)
    nb = min(args.nb, p.L * p.M)
    G = (cfg["n"] - 1) ** 2
    u = torch.empty((G, nb), dtype=torch.float64, device="cuda")
    B.usfft_sample_pde(ctx, B.pde_desc(cfg), p, 0, nb, u, nb)
    torch.cuda.synchronize()
    buf = (C.c_longlong * (16 * 32))()
    ctx.lib.usfft_debug_cl_probe(buf)
    v = [[buf[r * 32 + k] for k in range(32)] for r in range(16)]
    CS = 8 if cfg["n"] == 128 else 4
    for seq in ([20, 29, 30, 21, 22, 26, 27, 28, 25, 31, 23], list(range(14))):
        print("phase".ljust(20) + "".join(f"  cta{r:<5d}" for r in range(CS)))
        for a, b in zip(seq[:-1], seq[1:]):
            print(NAMES[b].ljust(20) + "".join(f"{v[r][b] - v[r][a]:9d}" for r in range(CS)))
        print("total".ljust(20) + "".join(f"{v[r][seq[-1]] - v[r][seq[0]]:9d}" for r in range(CS)))


if __name__ == "__main__":
    main()
