"""Host-side cost of one detection round (config 2, t = 5): wall time of every C-ABI call and
the device time of the round, to size launch / sync overheads.  python tools/round_host_profile.py"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2109_04131_b200 import binding as B
    sys.argv = [sys.argv[0]]
    import bench
    from usfft_inputs import config
    cfg = config(2)
    det, I_prev, kt = bench.setup_detector(cfg, 0, None, 5)
    det.timing = False
    n_prev, nJ = I_prev.shape[0], I_prev.shape[0] * kt.numel()
    calls = {}
    orig = {}
    for name in ("usfft_plan_round", "usfft_lattice", "usfft_sample_pde", "usfft_lattice_fft",
                 "usfft_detect_select", "usfft_detect_union", "usfft_resolve"):
        f = getattr(B, name)
        orig[name] = f

        def wrap(*a, _f=f, _n=name, **k):
            t0 = time.perf_counter()
            r = _f(*a, **k)
            calls[_n] = calls.get(_n, 0.0) + (time.perf_counter() - t0)
            return r
        setattr(B, name, wrap)
    import paper_2109_04131_b200.driver as D
    D.B = B
    for rep in range(3):
        calls.clear()
        flags = torch.zeros(nJ, dtype=torch.uint8, device="cuda")
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        det.round(2, 5, 100 + rep, I_prev, n_prev, kt, 100, flags, want_coef=True)
        e1.record()
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"rep {rep}: device {e0.elapsed_time(e1):.3f} ms, host {1e3 * (t1 - t0):.3f} ms; "
              + " ".join(f"{k[6:]}={1e3 * v:.3f}" for k, v in calls.items()))


if __name__ == "__main__":
    main()
