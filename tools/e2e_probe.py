#!/usr/bin/env python3
"""End-to-end step of the MBv1 pointwise stack through spcv_cu_spmm_into_host
(pinned host buffers, H2D | kernel | D2H inside every call), for sweeping the
host path's knobs (SPCV_HOST_CHUNK_MB, SPCV_HOST_RAMP: read once per process).

  SPCV_HOST_CHUNK_MB=24 python tools/e2e_probe.py [--images 256] [--steps 5]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_09723_b200 as sp  # noqa: E402
from paper_1911_09723_b200.workloads import CONFIGS, activation_of, make_layer_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    layers = CONFIGS["c2-b256"]["layers"]()
    data = [make_layer_data(L, args.images, 1000 * (i + 1)) for i, L in enumerate(layers)]
    items = []
    for d in data:
        L = d.layer
        a = torch.from_numpy(d.act).pin_memory()
        o = torch.empty((args.images, L.cout, L.h, L.w)).pin_memory()
        items.append((sp.DeviceBcsr(d.weights), a.numpy(), d.bias, activation_of(L.act), o.numpy(),
                      sp.MicrokernelConfig(n=L.block_h)))
    flops = sum(d.flops() for d in data)
    nbytes = sum(d.act.nbytes for d in data) + sum(it[4].nbytes for it in items)

    def step():
        for dw, a, b, fused, o, kc in items:
            sp.spmm_host_batched(dw, a, b, fused, o, kc)

    for _ in range(2):
        step()
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t0)
    best, med = min(ts), sorted(ts)[len(ts) // 2]
    print(f"chunk_mb={os.environ.get('SPCV_HOST_CHUNK_MB', 'default')} ramp={os.environ.get('SPCV_HOST_RAMP', '1')}: "
          f"median {med * 1e3:.2f} ms/step ({flops / med / 1e9:.1f} GFLOP/s, {nbytes / med / 1e9:.1f} GB/s over PCIe), "
          f"best {best * 1e3:.2f} ms")


if __name__ == "__main__":
    main()
