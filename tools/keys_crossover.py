"""Crossover of the two key kernels: k_kappa_grouped (usfft_lattice_keys) against k_kappa_tiled
(usfft_lattice_keys_product in a build with -DUSFFT_KEYS_TILED_ALWAYS=1) over
|J| at the shapes of configs 2 and 4.  python tools/keys_crossover.py"""
import os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2109_04131_b200 import _native, build

out = "/tmp/libusfft_tiled.so"
subprocess.run([build.NVCC, *build.FLAGS, "-DUSFFT_KEYS_TILED_ALWAYS=1", "-o", out, *build.sources()], cwd=build.SRC,
               check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
_native.LIB_PATH = out
import torch
from paper_2109_04131_b200 import binding as B

ctx = B.Context(0)
rng = np.random.default_rng(0)
for G, M, L, n1 in ((961, 401, 17, 65), (3969, 2017, 31, 129), (16129, 4001, 17, 65)):
    Mh = M // 2 + 1
    spectra = torch.randn((G, L, Mh, 2), dtype=torch.float64, device="cuda")
    for mult in ((0.55, 2) if M == 4001 else (2, 4, 8, 16, 32, 64)):
        n_prev = max(1, int(mult * Mh) // n1)
        t = 3
        I_prev = np.unique(rng.integers(-64, 65, size=(4 * n_prev, t - 1)), axis=0)[:n_prev]
        kt = np.arange(-(n1 // 2), n1 - n1 // 2)
        J = np.concatenate([np.repeat(I_prev, n1, axis=0), np.tile(kt, len(I_prev))[:, None]], axis=1)   # j = a n1 + c
        nJ = J.shape[0]
        z = rng.integers(1, M, size=(L, t))
        p = B.Plan(t, M, L, t, -1, z, np.zeros(t))
        bd = torch.as_tensor((J @ z.T % M).T, dtype=torch.int32, device="cuda").contiguous()   # [L][|J|]
        k = torch.empty((G, nJ), dtype=torch.float64, device="cuda")
        m = torch.zeros(1, dtype=torch.float64, device="cuda")
        res = {}
        for name, call in (("grouped", lambda: B.usfft_lattice_keys(ctx, p, G, spectra, bd, nJ, nJ, k, nJ, m)),
                           ("tiled", lambda: B.usfft_lattice_keys_product(ctx, p, G, spectra, bd, nJ, 0, nJ, n1, k, nJ, m))):
            call(); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(ctx.stream); call(); e1.record(ctx.stream); torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            res[name] = float(np.median(ts))
        print(f"G {G} M {M} L {L} |J| {nJ} = {nJ / Mh:.1f} (M/2+1): grouped {res['grouped']:.3f} ms, tiled {res['tiled']:.3f} ms", flush=True)
