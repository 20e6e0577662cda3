#!/usr/bin/env python3
"""PCIe bound of the e2e path: pinned-host copies of one c2-b256 step's bytes
(all layer inputs H2D, all outputs D2H), each direction alone and both
concurrently on two streams (best of 3). bench.py's `e2e` is compared with the
concurrent time.

  python tools/pcie_bound.py [--h2d-bytes B] [--d2h-bytes B]
"""
import argparse
import time

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--h2d-bytes", type=int, default=1978162432)   # c2-b256 step inputs (+bias)
    ap.add_argument("--d2h-bytes", type=int, default=2774532096)   # c2-b256 step outputs
    a = ap.parse_args()
    n_in, n_out = a.h2d_bytes // 4, a.d2h_bytes // 4
    hi = torch.empty(n_in, dtype=torch.float32).pin_memory()
    ho = torch.empty(n_out, dtype=torch.float32).pin_memory()
    di = torch.empty(n_in, device="cuda")
    do = torch.empty(n_out, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def best(fn, reps=3):
        t = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            t = min(t, time.perf_counter() - t0)
        return t * 1e3

    def both():
        with torch.cuda.stream(s1):
            di.copy_(hi, non_blocking=True)
        with torch.cuda.stream(s2):
            ho.copy_(do, non_blocking=True)

    h2d = best(lambda: di.copy_(hi, non_blocking=True))
    d2h = best(lambda: ho.copy_(do, non_blocking=True))
    bo = best(both)
    print(f"H2D {n_in * 4 / 1e9:.2f} GB {h2d:.1f} ms ({n_in * 4 / h2d / 1e6:.1f} GB/s); "
          f"D2H {n_out * 4 / 1e9:.2f} GB {d2h:.1f} ms ({n_out * 4 / d2h / 1e6:.1f} GB/s); "
          f"concurrent {bo:.1f} ms ({(n_in + n_out) * 4 / bo / 1e6:.1f} GB/s)")


if __name__ == "__main__":
    main()
