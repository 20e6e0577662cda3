#!/usr/bin/env python3
"""Run MobileNet-v1-1.0 forwards through spcv_cu_model_forward (for ncu / timing).

  python tools/prof_network.py [--images 256] [--reps 3] [--mode strict|fast] [--check 2]

Prints the median forward time; under ncu profile the last forward's kernels
(e.g. -s <launches per forward x (reps-1)>). --check compares the logits of the
first N images with the reference executor (oracle/_ref run_network).
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1911_09723_b200 as sp  # noqa: E402
from paper_1911_09723_b200 import netfile  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--images", type=int, default=256)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--mode", choices=["strict", "fast"], default="strict")
    ap.add_argument("--check", type=int, default=0)
    args = ap.parse_args()
    net = netfile.build_mbv1(1.0, 0.9, seed=11)
    blob = netfile.serialize(net)
    m = sp.DeviceModel(blob)
    rng = np.random.default_rng(100)
    xh = rng.uniform(-1, 1, (args.images, 224, 224, 3)).astype(np.float32)
    x = torch.from_numpy(xh).cuda()
    strict = args.mode == "strict"
    m.forward(x, strict)
    torch.cuda.synchronize()
    ts = []
    for _ in range(args.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        y = m.forward(x, strict)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"MBv1-1.0 x{args.images} {args.mode}: median {statistics.median(ts):.3f} ms "
          f"({args.images / statistics.median(ts) * 1e3:.0f} images/s)")
    if args.check:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as orc  # checker only

        want = orc.Ref().run_model(blob, xh[:args.check])
        got = y[:args.check].cpu().numpy()
        ok = np.array_equal(got.view(np.uint32), np.asarray(want, np.float32).reshape(got.shape).view(np.uint32))
        print(f"check {args.check} images vs reference run_network: {'bit-exact' if ok else 'MISMATCH'}")


if __name__ == "__main__":
    main()
