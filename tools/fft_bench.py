"""Lattice FFT alone (usfft_lattice_fft without keys) on config-shaped slabs: time per call (CUDA
events, after warm-up) and algorithmic HBM bytes (8 G L M read + 16 G L (M/2+1) written) per
second.  python tools/fft_bench.py"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2109_04131_b200 import binding as B
    ctx = B.Context(0)
    out = []
    for G, M, L in ((961, 401, 17), (3969, 2017, 17), (16129, 4001, 17)):
        p = B.Plan(3, M, L, 3, -1, np.ones((L, 3), dtype=np.int64), np.zeros(3))
        u = torch.randn((G, L * M), dtype=torch.float64, device="cuda")
        sp = torch.empty((G, L, M // 2 + 1, 2), dtype=torch.float64, device="cuda")
        for _ in range(2):
            B.usfft_lattice_fft(ctx, p, G, u, [0, L * M], None, 0, sp, None, None)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(ctx.stream)
            B.usfft_lattice_fft(ctx, p, G, u, [0, L * M], None, 0, sp, None, None)
            e1.record(ctx.stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        byt = 8 * G * L * M + 16 * G * L * (M // 2 + 1)
        out.append({"G": G, "M": M, "L": L, "ms": ms, "GBps": byt / ms / 1e6, "frac_hbm": byt / ms / 1e6 / 6550.7})
        print(json.dumps(out[-1]), flush=True)


if __name__ == "__main__":
    main()
