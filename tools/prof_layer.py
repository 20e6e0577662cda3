#!/usr/bin/env python3
"""Run one workload layer's SpMM kernel a few times (for ncu / quick timing).

  python tools/prof_layer.py --config c2-b256 --layer pw7[,pw8...] [--reps 5] [--mode fast]

Prints per-launch CUDA-event times; under ncu use -k regex:spmm_bcsr -s <warmups>.
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1911_09723_b200 as sp  # noqa: E402
from paper_1911_09723_b200.workloads import CONFIGS, activation_of, make_layer_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2-b256")
    ap.add_argument("--layer", default="pw7")
    ap.add_argument("--images", type=int, default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--mode", choices=["strict", "fast"], default="strict")
    ap.add_argument("--check", type=int, default=0,
                    help="compare the first N images with the CPU oracle (strict: bit-exact)")
    ap.add_argument("--adhoc", default=None,
                    help="K,M,H,W,sparsity,block_h,images: a synthetic layer instead of a config layer")
    args = ap.parse_args()
    if args.adhoc:
        from paper_1911_09723_b200.workloads import Layer
        K, M, H, W, sp_, bh, images = args.adhoc.split(",")
        L = Layer("adhoc", int(K), int(M), int(H), int(W), ("clamp", 0.0, float("inf")), -1.0, 1.0,
                  float(sp_), int(bh))
        args.images = int(images)
        run_layer(args, {"images": int(images)}, 0, L, "adhoc")
        return
    cfg = CONFIGS[args.config]
    layers = {L.name: (i, L) for i, L in enumerate(cfg["layers"]())}
    for name in args.layer.split(","):
        run_layer(args, cfg, *layers[name], name)


def run_layer(args, cfg, li, L, name):
    images = args.images or cfg["images"]
    d = make_layer_data(L, images, 1000 * (li + 1))
    dw = sp.DeviceBcsr(d.weights)
    import time
    t0 = time.time()
    kern = dw.kernel_for(images, L.h, L.w, args.mode == "strict")
    prep = time.time() - t0
    a = torch.from_numpy(d.act).cuda()
    b = torch.from_numpy(d.bias).cuda()
    o = torch.empty(images, L.cout, L.h, L.w, device="cuda")
    kc = sp.MicrokernelConfig(n=L.block_h, strict=args.mode == "strict")
    fused = activation_of(L.act)
    for _ in range(args.warmup):
        sp.spmm_batched_into(dw, a, b, fused, o, kc)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(200_000)  # the launch is queued before e0 runs: device time only
        e0.record()
        sp.spmm_batched_into(dw, a, b, fused, o, kc)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    us = statistics.median(ts)
    if args.check:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import Oracle  # checker only
        import numpy as np
        n = args.check
        got = o[:n].cpu().numpy()
        want = Oracle().spmm(d.weights, d.act[:n], d.bias, L.act, nthreads=os.cpu_count() or 1).reshape(got.shape)
        if args.mode == "strict":
            bad = int((got.view(np.uint32) != want.view(np.uint32)).sum())
        else:
            bad = int((np.abs(got - want) > 1e-4 * (1 + np.abs(want))).sum())
        print(f"{name} check {n} images: {'OK' if bad == 0 else f'{bad} MISMATCHES'}")
    print(f"{name} kernel={kern} (prep {prep:.1f}s) K={L.cin} M={L.cout} S={L.spatial} images={images} slots={dw.row_slots} "
          f"median {us:.1f} us  {d.flops() / us / 1e3:.0f} GFLOP/s  {d.alg_bytes() / us / 1e3:.0f} GB/s "
          f"(alg bytes {d.alg_bytes():.0f})")


if __name__ == "__main__":
    main()
