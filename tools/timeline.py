#!/usr/bin/env python3
"""Per-CTA phase timeline of one tile-kernel launch (needs the timeline build:
  make -C paper_1911_09723_b200/csrc VARIANT=tl VFLAGS=-DSPCV_TIMELINE
  SPCV_CU_LIB=paper_1911_09723_b200/lib/variants/libspcv_cu_tl.so python tools/timeline.py --config c5 --layer c5_s98

Every CTA records {SM, entry, tile staged (after the barrier), first / last warp
done, exit} with %globaltimer. Prints, per launch: kernel span, CTAs per SM,
and the mean time a CTA spends staging / computing / waiting for its slowest
warp / in its epilogue tail, plus per-SM busy fractions (how much of the kernel
span at least one CTA of the SM was in its compute phase)."""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_09723_b200 as sp  # noqa: E402
from paper_1911_09723_b200 import _capi  # noqa: E402
from paper_1911_09723_b200.workloads import CONFIGS, Layer, activation_of, make_layer_data  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--layer", default="c5_s98")
    ap.add_argument("--images", type=int, default=None)
    ap.add_argument("--adhoc", default=None, help="K,M,H,W,sparsity,block_h,images")
    args = ap.parse_args()
    lib = _capi.lib
    if not hasattr(lib, "spcvx_set_timeline"):
        try:
            lib.spcvx_set_timeline
        except AttributeError:
            sys.exit("this library was not built with -DSPCV_TIMELINE")
    lib.spcvx_set_timeline.argtypes = [ctypes.c_void_p]
    lib.spcvx_set_timeline.restype = None
    if args.adhoc:
        K, M, H, W, s, bh, images = args.adhoc.split(",")
        todo = [(Layer("adhoc", int(K), int(M), int(H), int(W), ("clamp", 0.0, float("inf")), -1.0, 1.0, float(s),
                       int(bh)), int(images))]
    else:
        cfg = CONFIGS[args.config]
        layers = {L.name: L for L in cfg["layers"]()}
        todo = [(layers[n], args.images or cfg["images"]) for n in args.layer.split(",")]
    for L, images in todo:
        d = make_layer_data(L, images, 1)
        dw = sp.DeviceBcsr(d.weights)
        a = torch.from_numpy(d.act).cuda()
        b = torch.from_numpy(d.bias).cuda()
        o = torch.empty(images, L.cout, L.h, L.w, device="cuda")
        kc = sp.MicrokernelConfig(n=L.block_h)
        fused = activation_of(L.act)
        for _ in range(3):  # first call autotunes
            sp.spmm_batched_into(dw, a, b, fused, o, kc)
        torch.cuda.synchronize()
        buf = torch.zeros(8 * 70000, dtype=torch.int64, device="cuda")
        lib.spcvx_set_timeline(ctypes.c_void_p(buf.data_ptr()))
        sp.spmm_batched_into(dw, a, b, fused, o, kc)
        torch.cuda.synchronize()
        lib.spcvx_set_timeline(None)
        t = buf.cpu().numpy().reshape(-1, 8)
        t = t[t[:, 1] != 0]
        t0 = t[:, 1].min()
        span = (t[:, 5].max() - t0) / 1e3
        sm = t[:, 0]
        entry, staged, first, last, exit_ = [(t[:, i] - t0) / 1e3 for i in (1, 2, 3, 4, 5)]
        print(f"{L.name}: K={L.cin} M={L.cout} S={L.spatial} x{images}, bh{L.block_h}, {L.sparsity:.0%}: "
              f"{len(t)} CTAs on {len(np.unique(sm))} SMs, kernel span {span:.1f} us")
        print(f"  per CTA (mean us): stage {np.mean(staged - entry):.2f}  compute(first warp done) "
              f"{np.mean(first - staged):.2f}  slowest warp +{np.mean(last - first):.2f}  "
              f"exit +{np.mean(exit_ - last):.2f}  lifetime {np.mean(exit_ - entry):.2f}")
        # per SM: fraction of the span with >= 1 CTA computing, and mean concurrent computing CTAs
        grid = np.linspace(0, span, 2000)
        busy, conc, resident = [], [], []
        for s in np.unique(sm):
            m = sm == s
            c = ((staged[m][:, None] <= grid[None, :]) & (grid[None, :] < last[m][:, None])).sum(0)
            r = ((entry[m][:, None] <= grid[None, :]) & (grid[None, :] < exit_[m][:, None])).sum(0)
            busy.append((c > 0).mean())
            conc.append(c.mean())
            resident.append(r.mean())
        print(f"  per SM: some CTA computing {np.mean(busy):.1%} of the span (min {np.min(busy):.1%}), "
              f"mean CTAs computing {np.mean(conc):.2f}, mean CTAs resident {np.mean(resident):.2f}; "
              f"last CTA starts at {entry.max():.1f} us, first exit at {exit_.min():.1f} us")


if __name__ == "__main__":
    main()
