"""Time usfft_eval (tensor-pipe DMMA vs CUDA-core FMA) on a config-5-like evaluation:
G nodes x n test points x |I| frequencies.  python tools/eval_bench.py [G n nI d]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2109_04131_b200 import binding as B
    G, n, nI, d = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (961, 100000, 313, 10)))
    ctx = B.Context(0)
    rng = np.random.default_rng(0)
    I = torch.as_tensor(rng.integers(-32, 33, size=(nI, d)) * (rng.random((nI, d)) < 0.3), dtype=torch.int16, device="cuda")
    C = torch.as_tensor(rng.standard_normal((G, nI, 2)), device="cuda")
    Y = torch.as_tensor(rng.random((d, n)), device="cuda")
    U = torch.empty((G, n), dtype=torch.float64, device="cuda")
    for mode in ("mma", "fma"):
        if mode == "fma":
            os.environ["USFFT_EVAL"] = "fma"
        for _ in range(2):
            B.usfft_eval(ctx, I, C, Y, U)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            B.usfft_eval(ctx, I, C, Y, U)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        flops = 2.0 * G * n * 2 * nI
        print(f"{mode}: {ms:.3f} ms, {flops / ms / 1e9:.2f} TFLOP/s (G={G} n={n} |I|={nI})")
        # the accuracy metric: real and imaginary parts (twice the products) + errors
        err = torch.empty((G, 3), dtype=torch.float64, device="cuda")
        B.usfft_eval_err(ctx, I, C, Y, U, err)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(5):
            B.usfft_eval_err(ctx, I, C, Y, U, err)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{mode} eval_err: {ms:.3f} ms, {2 * flops / ms / 1e9:.2f} TFLOP/s")


if __name__ == "__main__":
    main()
