"""Warm-process split of the detection time into Step 1 & 2a and Step 2 (config k):
python tools/detect_split.py [--config 2]"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    args = ap.parse_args()
    import torch
    from paper_2109_04131_b200.driver import Detector
    from usfft_inputs import config
    cfg = config(int(args.config) if args.config.isdigit() else args.config)
    det = Detector(cfg)
    det.run()
    torch.cuda.synchronize()
    for _ in range(2):
        t0 = time.perf_counter()
        I1d = det.step1()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        I, _ = det.step2(I1d)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        print(f"step1 {1e3 * (t1 - t0):.1f} ms ({cfg['d'] * cfg['r']} rounds), step2 {1e3 * (t2 - t1):.1f} ms, |I| {I.shape[0]}")


if __name__ == "__main__":
    main()
