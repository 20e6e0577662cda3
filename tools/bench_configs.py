#!/usr/bin/env python3
"""Per-config results for BASELINE.md §5 (one GPU): every BASELINE.json config,
every layer, cold-L2 and warm medians of 9 launches after 3 warm-ups
(BASELINE.md §2 "GPU timing"; the reference's median_time_ns scheme,
/root/reference/proj/src/bench.cpp:116-131), the binding roof per layer, a
strict-mode parity check of image 0 of every layer against the CPU oracle,
and the reference CPU kernel (oracle/_ref) on 1 thread and on all host cores.

  python tools/bench_configs.py [--configs c1,c2-b1,...] [--out profiles/r2_configs]

Writes <out>.json and <out>.md (the §5 table). CUDA events on the launch
stream behind a ~100 µs spin kernel (so host call overhead is not in the
device time; bench.py's e2e carries it); "cold" = the 126 MB L2 overwritten by a 252 MB fill before each timed
launch; "warm" = the same launch repeated back to back (inputs left in L2
when they fit).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1911_09723_b200.workloads import CONFIGS, make_layer_data  # noqa: E402

REPS, WARM = 9, 3
GATE_CYCLES = 200_000
L2 = 126 * 1024 * 1024


def roofs(d, hbm_gbs: float, f_clk: float, sms: int) -> dict:
    """Lower bounds on a layer's time (µs): HBM (algorithmic bytes at the
    measured copy bandwidth), the shared-memory gather (one 4 B activation per
    stored block per column, 128 B/clk/SM), and the strict FP32 issue roof
    (FMUL + FADD per product: 64 products/clk/SM)."""
    t_hbm = d.alg_bytes() / (hbm_gbs * 1e9) * 1e6
    nb = d.weights.nnz_blocks()
    cols = d.images * d.layer.spatial
    t_gather = nb * cols / (32.0 * sms * f_clk) * 1e6
    t_fp = d.nnz * cols / (64.0 * sms * f_clk) * 1e6
    bound = max((t_hbm, "hbm"), (t_gather, "gather"), (t_fp, "fp32"))
    return {"t_hbm_us": t_hbm, "t_gather_us": t_gather, "t_fp_us": t_fp, "binding": bound[1],
            "t_bound_us": bound[0]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2-b1,c2-b256,c3,c4,c5")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_configs"))
    ap.add_argument("--mode", choices=["strict", "fast"], default="strict")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()

    import paper_1911_09723_b200 as sp

    dev = 0
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    hbm, peak_kind = bench.peaks()
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    flush = torch.empty(2 * L2 // 4, dtype=torch.float32, device="cuda")
    orc = bench._oracle()
    oracle = orc.Oracle()
    threads = os.cpu_count() or 1
    # floor of this timing method: an empty-ish launch (a 4-byte fill) measured the same way
    tiny = torch.zeros(1, device="cuda")
    floor = []
    with torch.cuda.stream(stream):
        for _ in range(REPS):
            torch.cuda._sleep(GATE_CYCLES)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tiny.fill_(1.0)
            e1.record(stream)
            floor.append((e0, e1))
        stream.synchronize()
    floor_us = statistics.median(e0.elapsed_time(e1) * 1e3 for e0, e1 in floor)
    results = {"hbm_gbs": hbm, "peak_kind": peak_kind, "sms": sms, "configs": {},
               "timing_floor_us": floor_us,
               "cpu": {"model": bench.cpu_model(), "cores": threads,
                       "kind": "reference" if orc.have_ref() else "port"}}
    for cname in args.configs.split(","):
        cfg = CONFIGS[cname]
        layers = cfg["layers"]()
        images = cfg["images"]
        data = bench.gen_data(layers, images, 0)
        dev_layers = bench.upload(sp, data, images, dev, args.mode)
        rows = []
        with bench.ClockProbe(dev) as clk, torch.cuda.stream(stream):
            for d, (dw, a, b, o, fused, cfgk) in zip(data, dev_layers):
                def launch():
                    sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)

                for _ in range(WARM):
                    launch()
                stream.synchronize()
                times = {}
                for kind in ("cold", "warm"):
                    evs = []
                    for _ in range(REPS):
                        if kind == "cold":
                            flush.fill_(1.0)
                        # the stream waits ~100 us so the host has queued the launch
                        # before e0 runs: device time, not Python call overhead
                        torch.cuda._sleep(GATE_CYCLES)
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        launch()
                        e1.record(stream)
                        evs.append((e0, e1))
                    stream.synchronize()
                    times[kind] = statistics.median(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)
                # parity: image 0 in strict mode vs the oracle's matmul_reference
                L = d.layer
                if args.mode == "strict":
                    want = oracle.matmul_reference(d.dense, d.act[0].reshape(L.cin, -1), d.bias, L.act)
                    got = o[0].cpu().numpy().reshape(want.shape)
                    parity = "bit-exact" if np.array_equal(got.view(np.uint32), want.view(np.uint32)) \
                        else "MISMATCH"
                else:
                    parity = "n/a (fast)"
                rows.append({"layer": L.name, "K": L.cin, "M": L.cout, "S": L.spatial, "bh": L.block_h,
                             "sparsity": L.sparsity, "images": images, "nnz": d.nnz,
                             "kernel": dw.kernel_for(images, L.h, L.w, args.mode == "strict"),
                             "cold_us": times["cold"], "warm_us": times["warm"],
                             "flops": d.flops(), "alg_bytes": d.alg_bytes(), "parity": parity})
        f_clk = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
        for r, d in zip(rows, data):
            r.update(roofs(d, hbm, f_clk, sms))
            for kind in ("cold", "warm"):
                t = r[f"{kind}_us"]
                r[f"{kind}_gflops"] = r["flops"] / t / 1e3
                r[f"{kind}_gbs"] = r["alg_bytes"] / t / 1e3
                r[f"{kind}_hbm_frac"] = r[f"{kind}_gbs"] / hbm
                r[f"{kind}_frac_of_bound"] = r["t_bound_us"] / t
        # CPU: the reference spmm_into per (layer, image), 1 thread and all cores, on a bounded sample
        cpu = None
        if not args.no_cpu:
            n1 = 1
            nall = min(images, max(threads, 1))
            s1 = [make_layer_data(d.layer, n1, 1000 * (li + 1)) for li, d in enumerate(data)]
            _, fl1, t1 = bench.cpu_reference_run(s1, 3, 1, 1)
            cpu = {"single_thread_gflops": fl1 / statistics.median(t1) / 1e9,
                   "single_thread_sample": f"{n1} image x {len(data)} layer(s), median of 3"}
            if images > 1:
                sa = [make_layer_data(d.layer, nall, 1000 * (li + 1)) for li, d in enumerate(data)]
                _, fla, ta = bench.cpu_reference_run(sa, 3, 1, threads)
                cpu.update(all_core_gflops=fla / statistics.median(ta) / 1e9,
                           all_core_sample=f"{nall} images x {len(data)} layer(s), {threads} threads, median of 3")
        tot = {k: sum(r[f"{k}_us"] for r in rows) for k in ("cold", "warm")}
        flops = sum(r["flops"] for r in rows)
        byts = sum(r["alg_bytes"] for r in rows)
        results["configs"][cname] = {
            "images": images, "layers": rows, "cpu": cpu, "clocks": clk.summary(),
            "sum_cold_us": tot["cold"], "sum_warm_us": tot["warm"],
            "cold_gflops": flops / tot["cold"] / 1e3, "warm_gflops": flops / tot["warm"] / 1e3,
            "cold_gbs": byts / tot["cold"] / 1e3, "parity": ("bit-exact" if all(r["parity"] == "bit-exact" for r in rows)
                                                            else "see layers")}
        print(f"{cname}: cold {tot['cold']:.1f} us, warm {tot['warm']:.1f} us, "
              f"{flops / tot['cold'] / 1e3:.0f} GFLOP/s cold", file=sys.stderr, flush=True)
        del dev_layers
        torch.cuda.empty_cache()
    json.dump(results, open(args.out + ".json", "w"), indent=1)
    open(args.out + ".md", "w").write(markdown(results))
    print(markdown(results))


def markdown(res) -> str:
    out = ["| Config | layer | GPUs | t cold / warm (µs) | GFLOP/s (2·nnz·N) cold | GB/s (B_alg) cold | "
           "% HBM roof cold | binding roof (bound µs) | % of binding roof cold | parity | kernel |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for cname, c in res["configs"].items():
        for r in c["layers"]:
            out.append(f"| {cname} | {r['layer']} ({r['K']}→{r['M']} @{r['S']}, bh{r['bh']}, "
                       f"{int(round(r['sparsity'] * 100))}%, ×{r['images']}) | 1 | "
                       f"{r['cold_us']:.1f} / {r['warm_us']:.1f} | {r['cold_gflops']:.0f} | {r['cold_gbs']:.0f} | "
                       f"{100 * r['cold_hbm_frac']:.1f} | {r['binding']} ({r['t_bound_us']:.1f}) | "
                       f"{100 * r['cold_frac_of_bound']:.0f} | {r['parity']} | {r['kernel']} |")
    out.append("")
    out.append(f"Timing floor of this method (a 4-byte fill kernel timed the same way): "
               f"{res.get('timing_floor_us', float('nan')):.1f} µs; CUDA event resolution on this GPU is 2.048 µs.")
    out.append("")
    out.append(f"CPU = the reference `spmm_into` (oracle/_ref, {res['cpu']['kind']}) on "
               f"{res['cpu']['model']} ({res['cpu']['cores']} threads).")
    out.append("")
    out.append("| Config | GPUs | Σ t cold / warm (µs) | GFLOP/s cold / warm | GB/s cold | parity | "
               "CPU 1-thread GFLOP/s | CPU all-core GFLOP/s (cores) |")
    out.append("|---|---|---|---|---|---|---|---|")
    for cname, c in res["configs"].items():
        cpu = c["cpu"] or {}
        allc = cpu.get("all_core_gflops")
        out.append(f"| {cname} | 1 | {c['sum_cold_us']:.1f} / {c['sum_warm_us']:.1f} | "
                   f"{c['cold_gflops']:.0f} / {c['warm_gflops']:.0f} | {c['cold_gbs']:.0f} | {c['parity']} | "
                   f"{cpu.get('single_thread_gflops', float('nan')):.2f} | "
                   f"{(f'{allc:.1f} ({res['cpu']['cores']})' if allc else 'batch 1: 1 thread only')} |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    main()
