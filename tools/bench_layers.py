#!/usr/bin/env python3
"""GPU `bench-layers` in the reference's CSV schema.

Emits exactly the 11 columns of /root/reference/proj/src/bench.cpp:428-445
(layer_index,kind,cout,cin,spatial,sparsity,block_h,variant,median_ns,
achieved_gflops,effective_gflops) with `%.17g` doubles, so downstream
plotting of the reference's `spcv bench-layers --csv` output works unchanged.
Rows per sparse pointwise layer: variant `b200-strict` (bit-exact kernel),
`b200-fast` (FFMA) and `dense` (cuBLAS fp32 on the unpruned weights), like the
reference's per-variant rows plus its dense row (bench.cpp:195-227).
Timing follows median_time_ns (bench.cpp:116-131): W warm-ups, R (odd) timed
runs, median — here with CUDA events. achieved = 2*nnz*S*images/t,
effective = 2*M*K*S*images/t (bench.cpp:211-212).

  python tools/bench_layers.py --arch mbv1 --images 1 --csv out.csv
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CSV_HEADER = ("layer_index,kind,cout,cin,spatial,sparsity,block_h,variant,median_ns,"
              "achieved_gflops,effective_gflops")


def fmt(v: float) -> str:
    return "%.17g" % v


def rows_to_csv(rows) -> str:
    out = [CSV_HEADER]
    for r in rows:
        out.append(",".join([str(r["layer_index"]), r["kind"], str(r["cout"]), str(r["cin"]),
                             str(r["spatial"]), fmt(r["sparsity"]), str(r["block_h"]), r["variant"],
                             fmt(r["median_ns"]), fmt(r["achieved_gflops"]),
                             fmt(r["effective_gflops"])]))
    return "\n".join(out) + "\n"


def main():
    import torch

    import paper_1911_09723_b200 as sp
    from paper_1911_09723_b200.workloads import activation_of, make_layer_data, mbv1_pointwise, mbv2_pointwise

    ap = argparse.ArgumentParser()
    ap.add_argument("--arch", choices=["mbv1", "mbv2"], default="mbv1")
    ap.add_argument("--sparsity", type=float, default=None)
    ap.add_argument("--images", type=int, default=1)
    ap.add_argument("--runs", type=int, default=9)
    ap.add_argument("--warmups", type=int, default=3)
    ap.add_argument("--csv", default=None)
    a = ap.parse_args()
    if a.runs < 3 or a.runs % 2 == 0:
        raise SystemExit("run count must be odd and at least 3 (bench.cpp:118)")
    layers = mbv1_pointwise(a.sparsity or 0.9) if a.arch == "mbv1" else mbv2_pointwise(a.sparsity or 0.85)

    def median_ns(fn):
        for _ in range(a.warmups):
            fn()
        ts = []
        for _ in range(a.runs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e6)
        return statistics.median(ts)

    rows = []
    for li, L in enumerate(layers):
        d = make_layer_data(L, a.images, 1000 * (li + 1))
        dw = sp.DeviceBcsr(d.weights)
        act = torch.from_numpy(d.act).cuda()
        bias = torch.from_numpy(d.bias).cuda()
        out = torch.empty(a.images, L.cout, L.h, L.w, device="cuda")
        fused = activation_of(L.act)
        cols = a.images * L.spatial
        dense_flops = 2.0 * L.cout * L.cin * cols
        base = dict(layer_index=L.net_index, kind="pointwise", cout=L.cout, cin=L.cin,
                    spatial=L.spatial)
        for variant, strict in (("b200-strict", True), ("b200-fast", False)):
            cfg = sp.MicrokernelConfig(n=L.block_h, strict=strict)
            ns = median_ns(lambda: sp.spmm_batched_into(dw, act, bias, fused, out, cfg))
            rows.append(dict(base, sparsity=L.sparsity, block_h=L.block_h, variant=variant,
                             median_ns=ns, achieved_gflops=2.0 * d.nnz * cols / ns,
                             effective_gflops=dense_flops / ns))
        # dense row: the unpruned (He-style random) matrix, as bench.cpp:216-227
        wd = torch.randn(L.cout, L.cin, device="cuda") * 0.1
        ns = median_ns(lambda: sp.dense_gemm_batched_into(wd, act, bias, fused, out))
        rows.append(dict(base, sparsity=0.0, block_h=1, variant="dense", median_ns=ns,
                         achieved_gflops=dense_flops / ns, effective_gflops=dense_flops / ns))
    text = rows_to_csv(rows)
    if a.csv:
        open(a.csv, "w").write(text)
    sys.stdout.write(text)


if __name__ == "__main__":
    main()
