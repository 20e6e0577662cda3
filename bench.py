#!/usr/bin/env python3
"""Benchmark of the B200 sparse 1x1-conv SpMM (the north-star path).

Default workload (BASELINE.json configs[1]): the 13 MobileNet-v1-1.0 pointwise
layers at 224x224, 90% unstructured sparsity, ReLU6, fp32, 256 images per GPU
(weak scaling: each rank runs its own 256-image shard, no collective on the
data path). One step = one pass of all 13 layers over the rank's batch.

Metric (BASELINE.json): effective GFLOP/s = 2*nnz*N / t summed over layers
(reference convention, /root/reference/proj/src/bench.cpp:211), plus
algorithmic HBM GB/s against the measured peak.

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

Rank 0 prints ONE JSON line on stdout; details go to stderr.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1911_09723_b200.dist import Dist, shard  # noqa: E402
from paper_1911_09723_b200.workloads import CONFIGS, activation_of, make_layer_data  # noqa: E402

WORKLOAD_DESC = {
    "c2-b256": "MobileNet-v1-1.0 pointwise stack @224 (13 layers), 90% unstructured, ReLU6",
    "c2-b1": "MobileNet-v1-1.0 pointwise stack @224 (13 layers), 90% unstructured, ReLU6",
    "c1": "single 128x128 sparse 1x1 conv @28x28, 80% unstructured, ReLU",
    "c3": "512x512 @14x14, block 4/2/1 x1, sparsity 70-95%, ReLU",
    "c4": "MobileNet-v2-1.0 1x1 convs @224, 85% unstructured, ReLU6/linear",
    "c5": "1024x1024 @7x7, Beta(2,8)-skewed rows, sparsity 70-98%, ReLU",
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ------------------------------------------------------------- clock probe
class ClockProbe:
    """Samples SM clock and throttle reasons via NVML every 10 ms while running."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], 0, False
        self.max_mhz = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - box-specific
            log(f"clock probe unavailable: {e}")
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            self._stop.wait(0.01)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml_unavailable"], "samples": 0}
        reasons = [n for b, n in self.REASONS.items() if self.reasons & b and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU reference
def cpu_reference_run(layers_data, steps: int, warmup: int, threads: int):
    """Reference spmm_into (oracle/_ref, else the oracle port) on host cores.
    Every (layer, image) pair is one spmm_into call; `threads` host threads
    pull them longest-first (oracle/ref_shim.cpp: ref_bench_layers)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc  # CPU baseline leg only

    flops = sum(d.flops() for d in layers_data)
    if orc.have_ref():
        ref = orc.Ref()
        times = ref.bench_layers([(d.weights, d.act, d.bias, d.layer.act) for d in layers_data],
                                 threads, warmup, steps)
        return "reference", flops, times
    port = orc.Oracle()
    times = []
    for s in range(warmup + steps):
        t0 = time.perf_counter()
        for d in layers_data:
            port.spmm(d.weights, d.act, d.bias, d.layer.act, nthreads=threads)
        if s >= warmup:
            times.append(time.perf_counter() - t0)
    return "port", flops, times


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="c2-b256", choices=sorted(CONFIGS))
    ap.add_argument("--images", type=int, default=None, help="images per GPU (default: config's)")
    ap.add_argument("--global-batch", type=int, default=None,
                    help="strong scaling: shard this many images over the ranks instead")
    ap.add_argument("--mode", choices=["strict", "fast"], default="strict")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dense", action="store_true", help="skip the cuBLAS dense fp32 baseline")
    ap.add_argument("--cpu-images", type=int, default=None, help="CPU baseline sample, images")
    ap.add_argument("--layers-json", default=None, help="write per-layer results here")
    ap.add_argument("--no-alt", action="store_true",
                    help="skip the other arithmetic mode and the CUDA-graph replay (profiling runs)")
    ap.add_argument("--no-network", action="store_true",
                    help="skip the whole-network (device executor) measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup < 3 is not allowed by the timing rules; using 3")
        args.warmup = 3

    cfg = CONFIGS[args.config]
    layers = cfg["layers"]()
    images = args.images or cfg["images"]
    hbm_peak, peak_kind = peaks()

    if args.impl == "reference":
        return run_reference(args, layers, images)

    import torch

    # SPCV_DIST_BACKEND=gloo runs the N>1 code path with ranks sharing a GPU
    # (a functional check on a one-GPU box; NCCL refuses two ranks per GPU)
    dist = Dist(os.environ.get("SPCV_DIST_BACKEND", "nccl"))
    dev = dist.local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(dev)
    import paper_1911_09723_b200 as sp

    scaling = "weak"
    if args.global_batch:  # strong scaling: contiguous image shard per rank
        b0, b1 = shard(args.global_batch, dist.world, dist.rank)
        images, scaling = b1 - b0, "strong"

    # ---- data: weights identical on every rank, activations per-rank shard
    t0 = time.time()
    data = []
    for li, L in enumerate(layers):
        d = make_layer_data(L, images, 1000 * (li + 1) + dist.rank)
        w = make_layer_data(L, 1, 1000 * (li + 1), act=False)  # weights: rank-independent seed
        d.weights, d.dense, d.bias = w.weights, w.dense, w.bias
        data.append(d)
    log(f"[rank {dist.rank}] generated {len(layers)} layers x {images} images in {time.time() - t0:.1f}s")

    stream = torch.cuda.Stream(dev)
    mode_cfg = {}
    dev_layers = []
    for d in data:
        dw = sp.DeviceBcsr(d.weights)
        a = torch.from_numpy(d.act).to(dev)
        o = torch.empty((images, d.layer.cout, d.layer.h, d.layer.w), device=dev)
        b = torch.from_numpy(d.bias).to(dev)
        cfgk = sp.MicrokernelConfig(n=d.layer.block_h, strict=(args.mode == "strict"))
        dev_layers.append((dw, a, b, o, activation_of(d.layer.act), cfgk))
        mode_cfg[d.layer.name] = dw.row_slots
    torch.cuda.synchronize()

    def step(evs=None):
        for li, (dw, a, b, o, fused, cfgk) in enumerate(dev_layers):
            if evs is not None:
                evs[li][0].record(stream)
            sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)
            if evs is not None:
                evs[li][1].record(stream)

    flops_step = sum(d.flops() for d in data)
    bytes_step = sum(d.alg_bytes() for d in data)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        nl = len(dev_layers)
        lev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(nl)]
               for _ in range(args.steps)]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier(dev)
        torch.cuda.synchronize()
        launches0 = sp.launch_count()
        with ClockProbe(dev) as clk:
            start.record(stream)
            for k in range(args.steps):
                step()
            end.record(stream)
            torch.cuda.synchronize()
        launches = sp.launch_count() - launches0
        dist.barrier(dev)
        # per-layer breakdown: a separate pass with events around every launch
        # (kept out of the headline region: the event records add gaps)
        for k in range(args.steps):
            step(lev[k])
        torch.cuda.synchronize()
    ms_local = start.elapsed_time(end)
    ms_total = dist.max(ms_local, device=torch.device("cuda", dev))
    ms_step = ms_total / args.steps

    # The same step replayed as one CUDA graph (the 13 launches captured once):
    # launch overhead out of the way, which matters for the batch-1 configs.
    # Every rank reaches the same collectives whether or not its capture works
    # (a failure is reported as -1 and the max over ranks tells every rank).
    graph = None
    if not args.no_alt:
        ms_local, err = -1.0, ""
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(stream):
                step()  # every kernel variant exists before capture
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=stream):
                    step()
                g.replay()
                torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001 - reported, the eager number stands
            g, err = None, repr(e)[:200]
        flag = 1.0 if g is not None else -1.0
        ok = -dist.max(-flag, device=torch.device("cuda", dev)) > 0  # min over ranks: all captured
        if ok:
            with torch.cuda.stream(stream):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                dist.barrier(dev)
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(args.steps):
                    g.replay()
                e1.record(stream)
                torch.cuda.synchronize()
            ms_local = e0.elapsed_time(e1)
        ms_graph = dist.max(ms_local, device=torch.device("cuda", dev)) / args.steps if ok else -1.0
        if ok:
            graph = {"ms_per_step": round(ms_graph, 4),
                     "value": round(dist.sum(flops_step, device=torch.device("cuda", dev)) / (ms_graph * 1e-3) / 1e9, 3),
                     "how": "torch.cuda.CUDAGraph capture of one step (13 spcv_cu_spmm_into launches), replayed"}
        else:
            graph = {"unavailable": err or "capture failed on another rank"}
        del g

    # The other arithmetic mode on the same packed weights (reported beside the
    # headline, which is the mode selected by --mode): strict = bit-exact,
    # fast = FFMA within the north_star tolerance.
    other = "fast" if args.mode == "strict" else "strict"
    alt_cfgs = [sp.MicrokernelConfig(n=c.n, strict=(other == "strict")) for (_, _, _, _, _, c) in dev_layers]

    def step_alt():
        for (dw, a, b, o, fused, _), cfgk in zip(dev_layers, alt_cfgs):
            sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)

    ms_alt = float("nan")
    if not args.no_alt:
        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                step_alt()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier(dev)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(args.steps):
                step_alt()
            e1.record(stream)
            torch.cuda.synchronize()
        ms_alt = dist.max(e0.elapsed_time(e1), device=torch.device("cuda", dev)) / args.steps

    # per-layer kernel times (events on the launch stream, averaged over steps)
    per_layer = []
    for li, d in enumerate(data):
        us = statistics.mean(lev[k][li][0].elapsed_time(lev[k][li][1]) for k in range(args.steps)) * 1e3
        per_layer.append(dict(name=d.layer.name, K=d.layer.cin, M=d.layer.cout, S=d.layer.spatial,
                              bh=d.layer.block_h, nnz=d.nnz, row_slots=mode_cfg[d.layer.name],
                              us=us, gflops=d.flops() / us / 1e3, gbs=d.alg_bytes() / us / 1e3,
                              hbm_frac=d.alg_bytes() / us / 1e3 / hbm_peak,
                              alg_bytes=d.alg_bytes(), flops=d.flops(),
                              kernel=("spcv_jit" if dev_layers[li][0].kernel(args.mode == "strict") == "jit"
                                      else "spmm_bcsr_kernel")))
    tot_us = sum(p["us"] for p in per_layer)
    for p in per_layer:
        p["share"] = p["us"] / tot_us
    dom = max(per_layer, key=lambda p: p["us"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom["name"])
        except Exception:
            traffic = None

    # aggregate GFLOP/s: every rank's FLOPs over the max-over-ranks time
    flops_all = dist.sum(flops_step, device=torch.device("cuda", dev))
    value = flops_all / (ms_step * 1e-3) / 1e9
    if dist.rank == 0:
        log(f"{'layer':6s} {'K':>5s} {'M':>5s} {'S':>6s} {'slots':>5s} {'us':>9s} {'GFLOP/s':>9s} "
            f"{'GB/s':>8s} {'HBM%':>6s} {'share':>6s}")
        for p in per_layer:
            log(f"{p['name']:6s} {p['K']:5d} {p['M']:5d} {p['S']:6d} {p['row_slots']:5d} {p['us']:9.1f} "
                f"{p['gflops']:9.0f} {p['gbs']:8.0f} {100 * p['hbm_frac']:6.1f} {100 * p['share']:6.1f}")
        log(f"step {ms_step:.3f} ms; layer kernels sum {tot_us / 1e3:.3f} ms; "
            f"{value:.0f} GFLOP/s aggregate over {dist.world} GPU(s)")
        if args.layers_json:
            json.dump(per_layer, open(args.layers_json, "w"), indent=1)

    # ---- dense fp32 baseline (reference dense_gemm_into, bench.cpp:216-227): the
    # same layers with dense weights through cuBLAS SGEMM (pedantic fp32)
    dense = None
    if not args.no_dense:
        dws = [torch.from_numpy(d.dense).to(dev) for d in data]
        dcfg = sp.MicrokernelConfig()

        def step_dense(evs=None):
            for li, ((_, a, b, o, fused, _), w) in enumerate(zip(dev_layers, dws)):
                if evs is not None:
                    evs[li][0].record(stream)
                sp.dense_gemm_batched_into(w, a, b, fused, o, dcfg, stream=stream)
                if evs is not None:
                    evs[li][1].record(stream)

        with torch.cuda.stream(stream):
            for _ in range(args.warmup):
                step_dense()
            dsteps = max(1, min(args.steps, 5))
            dev_ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in dws]
                      for _ in range(dsteps)]
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier(dev)
            torch.cuda.synchronize()
            e0.record(stream)
            for k in range(dsteps):
                step_dense(dev_ev[k])
            e1.record(stream)
            torch.cuda.synchronize()
        ms_dense = dist.max(e0.elapsed_time(e1), device=torch.device("cuda", dev)) / dsteps
        dense_flops = sum(2.0 * d.layer.cout * d.layer.cin * d.images * d.layer.spatial for d in data)
        for li, p in enumerate(per_layer):
            p["dense_us"] = statistics.mean(dev_ev[k][li][0].elapsed_time(dev_ev[k][li][1])
                                            for k in range(dsteps)) * 1e3
        dense = {"ms_per_step": round(ms_dense, 4),
                 "dense_gflops": round(dense_flops * dist.world / (ms_dense * 1e-3) / 1e9, 1),
                 "sparse_effective_gflops": round(dense_flops * dist.world / (ms_step * 1e-3) / 1e9, 1),
                 "sparse_speedup_vs_dense": round(ms_dense / ms_step, 3),
                 "per_layer_speedup": {p["name"]: round(p["dense_us"] / p["us"], 2) for p in per_layer},
                 "how": "cuBLAS SGEMM strided-batched (CUBLAS_PEDANTIC_MATH) + bias/clamp epilogue, "
                        f"same inputs, {dsteps} steps"}
        del dws
        with torch.cuda.stream(stream):
            step()  # restore the sparse outputs for the e2e check below
        torch.cuda.synchronize()
        if dist.rank == 0:
            log(f"dense fp32 baseline: {ms_dense:.3f} ms/step; sparse speedup {ms_dense / ms_step:.2f}x")

    # ---- end-to-end: the host-buffer C-ABI call (H2D + kernel + D2H per layer)
    e2e = None
    if not args.no_e2e:
        host = []
        for d in data:
            a = torch.from_numpy(d.act).pin_memory()
            o = torch.empty((images, d.layer.cout, d.layer.h, d.layer.w)).pin_memory()
            host.append((a.numpy(), o.numpy()))
        h2d = sum(d.act.nbytes + d.bias.nbytes for d in data)
        d2h = sum(o.nbytes for _, o in host)

        def e2e_step():
            for (dw, _, _, _, fused, cfgk), d, (a, o) in zip(dev_layers, data, host):
                sp.spmm_host_batched(dw, a, d.bias, fused, o, cfgk)

        for _ in range(args.warmup):
            e2e_step()
        dist.barrier(dev)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        dt = time.perf_counter() - t0
        dt = dist.max(dt, device=torch.device("cuda", dev))
        e2e = {"value": round(flops_all / (dt / args.steps) / 1e9, 3),
               "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(dt / args.steps * 1e3, 3),
               "path": "spcv_cu_spmm_into_host per layer (pinned host buffers; image chunks pipelined H2D|kernel|D2H on 3 streams)"}
        # e2e outputs must equal the device path's outputs (re-run one step of
        # the headline mode: the alternate-mode timing overwrote the outputs)
        with torch.cuda.stream(stream):
            step()
        torch.cuda.synchronize()
        for (_, _, _, o_dev, _, _), (_, o) in zip(dev_layers, host):
            if not np.array_equal(o_dev.cpu().numpy().view(np.uint32), o.view(np.uint32)):
                raise SystemExit("e2e output differs from the device-path output")

    # ---- the whole network on the device (run_network: entry conv, depthwise,
    # pooling, sparse 1x1 layers, classifier), informational beside the headline
    network = None
    if not args.no_network:
        network = bench_network(args, dev, stream, dist, images)

    # ---- CPU baseline (rank 0, N=1 only), a bounded sample of the same workload
    cpu = None
    if dist.world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        n_img = min(args.cpu_images or images, images)
        sample = data
        if n_img < images:
            sample = [make_layer_data(d.layer, n_img, 1000 * (li + 1)) for li, d in enumerate(data)]
        kind, flops, times = cpu_reference_run(sample, 3, 1, threads)
        # the reference's own concurrency model (one thread), on an 8-image slice
        s1 = [make_layer_data(d.layer, min(8, images), 1000 * (li + 1)) for li, d in enumerate(data)]
        _, flops1, times1 = cpu_reference_run(s1, 3, 1, 1)
        cpu_model = ""
        try:
            for line in open("/proc/cpuinfo"):
                if line.startswith("model name"):
                    cpu_model = line.split(":", 1)[1].strip()
                    break
        except OSError:
            pass
        cpu = {"value": round(flops / statistics.median(times) / 1e9, 3), "unit": "GFLOP/s",
               "cores": threads, "kind": kind, "cpu_model": cpu_model,
               "single_thread": {"value": round(flops1 / statistics.median(times1) / 1e9, 3),
                                 "sample": f"{min(8, images)} images x all layers, 1 thread, median of 3"},
               "sample": f"{n_img} image(s) x all {len(layers)} layers of {args.config} "
                         f"(= {'the full step' if n_img == images else 'a slice of the step'}), "
                         f"(layer,image) spmm_into units over {threads} threads, median of 3 passes "
                         f"after 1 warm-up: {statistics.median(times):.3f}s/pass"}

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_sum = clk.summary()
    f_clk = (clk_sum.get("sm_mhz") or clk_sum.get("sm_max_mhz") or 1965.0) * 1e6
    gather_roof = sms * 64 * f_clk / 1e12  # TFLOP/s
    if dist.rank == 0:
        roofline = {"bound": "hbm", "achieved": round(dom["gbs"], 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(dom["gbs"] / hbm_peak, 4), "traffic": traffic,
                    "kernel": f"{dom.get('kernel', 'tile')} [{dom['name']}: {dom['K']}->{dom['M']} @S={dom['S']}]",
                    "peak_kind": peak_kind,
                    "alg_bytes_per_launch": dom["alg_bytes"], "avg_launch_us": round(dom["us"], 2),
                    "share_of_step": round(dom["share"], 3),
                    "step_hbm_frac": round(bytes_step / (ms_step * 1e-3) / 1e9 / hbm_peak, 4),
                    "gather_roof_tflops": round(gather_roof, 2),
                    # SURVEY.md §8d "Cap": the best HBM fraction the binding roof allows for
                    # this layer (t_HBM / max(t_HBM, t_gather), gather roof x block height)
                    "attainable_frac": round(min(1.0, (dom["alg_bytes"] / (hbm_peak * 1e9)) /
                                                 max(dom["alg_bytes"] / (hbm_peak * 1e9),
                                                     dom["flops"] / (gather_roof * 1e12 * dom["bh"]))), 4),
                    "frac_of_attainable": round((dom["gbs"] / hbm_peak) / min(1.0, (dom["alg_bytes"] / (hbm_peak * 1e9)) /
                                                max(dom["alg_bytes"] / (hbm_peak * 1e9),
                                                    dom["flops"] / (gather_roof * 1e12 * dom["bh"]))), 4),
                    "gather_frac": round(dom["gflops"] / 1e3 / gather_roof, 4),
                    # every layer of the step against its roofs: the tile kernel is bound by
                    # the lower of HBM and the shared-memory gather; the weight-specialised
                    # (spcv_jit) kernels gather nothing (activations in registers): HBM only
                    "layers": {p["name"]: {
                        "kernel": p["kernel"], "us": round(p["us"], 1),
                        "bound": "hbm" if p["kernel"] == "spcv_jit" or p["alg_bytes"] / (hbm_peak * 1e9) >=
                                 p["flops"] / (gather_roof * 1e12 * p["bh"]) else "gather",
                        "hbm_frac": round(p["hbm_frac"], 4),
                        "gather_frac": (None if p["kernel"] == "spcv_jit" else
                                        round(p["gflops"] / 1e3 / (gather_roof * p["bh"]), 4))}
                        for p in per_layer},
                    "step_gather_frac": round(value / 1e3 / dist.world / gather_roof, 4),
                    "note": "achieved = SURVEY.md §8d algorithmic bytes / CUDA-event launch time. "
                            "Layers with AI > ~2.9 FLOP/B are bound by the shared-memory gather roof "
                            "(one 4 B activation per stored block per column at 128 B/clk/SM: "
                            "SMs x 64 FLOP/clk x SM clock), not HBM; gather_frac is against that roof "
                            "at the clock measured during the run"}
        line = {
            "metric": "SpMM effective GFLOP/s (2*nnz*N)", "value": round(value, 3),
            "unit": "GFLOP/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE config shapes)",
            "config": {"workload": f"{args.config}: {WORKLOAD_DESC[args.config]}",
                       "images_per_gpu": images,
                       "global_batch": args.global_batch or images * dist.world,
                       "mode": args.mode, "parallelism": f"dp{dist.world} (image shards, no collective)",
                       "l2": f"inputs larger than L2: {bytes_step / 1e9:.2f} GB touched per step "
                             f"per GPU vs 126 MB L2, no explicit flush"},
            "hbm_gbs": round(bytes_step / (ms_step * 1e-3) / 1e9, 1),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "dense_baseline": dense,
            "network": network, "graph": graph,
            "gpu_launches": launches, "clocks": clk.summary(),
            "modes": {args.mode: {"value": round(value, 3), "ms_per_step": round(ms_step, 4)},
                      other: ({"value": round(flops_all / (ms_alt * 1e-3) / 1e9, 3),
                               "ms_per_step": round(ms_alt, 4)} if ms_alt == ms_alt else None),
                      "note": "strict = bit-exact vs the reference CPU kernel (default); "
                              "fast = FFMA, within the north_star nnz-scaled 1e-5 tolerance"},
        }
        print(json.dumps(line), flush=True)
    dist.close()


def bench_network(args, dev, stream, dist, batch):
    """MobileNet-v1-1.0 @224 as an SPCV model file (netfile.py: the reference's
    builder / default_plan / serializer restated, seeded synthetic weights),
    run end to end by spcv_cu_model_forward on `batch` images per GPU. Sparse
    strict and fast, the densified network (dense 1x1 via cuBLAS, fast), and
    batch-1 latency; CUDA events on the launch stream, max over ranks."""
    import torch

    import paper_1911_09723_b200 as sp
    from paper_1911_09723_b200 import netfile

    net = netfile.build_mbv1(1.0, 0.9, seed=11)
    blob = netfile.serialize(net)
    m = sp.DeviceModel(blob)
    md = sp.DeviceModel(netfile.serialize(netfile.densify(net)))
    rng = np.random.default_rng(100 + dist.rank)
    x = torch.from_numpy(rng.uniform(-1, 1, (batch, 224, 224, 3)).astype(np.float32)).to(dev)

    def timed(model, strict, inp, steps):
        with torch.cuda.stream(stream):
            for _ in range(max(2, args.warmup)):
                model.forward(inp, strict, stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier(dev)
            torch.cuda.synchronize()
            n0 = sp.launch_count()
            e0.record(stream)
            for _ in range(steps):
                model.forward(inp, strict, stream)
            e1.record(stream)
            torch.cuda.synchronize()
            launches = (sp.launch_count() - n0) // steps
        return dist.max(e0.elapsed_time(e1), device=torch.device("cuda", dev)) / steps, launches

    steps = max(3, min(args.steps, 10))
    ms_strict, launches = timed(m, True, x, steps)
    ms_fast, _ = timed(m, False, x, steps)
    ms_dense, _ = timed(md, False, x, steps)
    ms_b1, _ = timed(m, True, x[:1], 20)
    # batch-1 latency with the forward's launches captured once as a CUDA graph
    ms_b1_graph = None
    try:
        x1 = x[:1].clone()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            m.forward(x1, True, stream)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=stream):
                y1 = m.forward(x1, True, stream)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(50):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
        ms_b1_graph = round(e0.elapsed_time(e1) / 50, 4)
        del g, y1
    except Exception as e:  # noqa: BLE001
        log(f"network graph capture unavailable: {e!r}"[:200])
    log(f"network MBv1-1.0 x{batch}: strict {ms_strict:.3f} ms, fast {ms_fast:.3f} ms, "
        f"dense(cuBLAS) {ms_dense:.3f} ms, batch-1 latency {ms_b1:.3f} ms")
    out = {"model": "MobileNet-v1-1.0 @224x224x3: entry conv, 13 depthwise + 13 sparse 1x1 (90%, "
                    "4x1 blocks from pw12: the reference's default_plan), pool, dense classifier",
           "images_per_gpu": batch, "mode": "strict",
           "images_per_s": round(batch * dist.world / (ms_strict * 1e-3), 1),
           "ms_per_batch": round(ms_strict, 3), "fast_ms_per_batch": round(ms_fast, 3),
           "dense_cublas_ms_per_batch": round(ms_dense, 3),
           "sparse_speedup_vs_dense": round(ms_dense / ms_fast, 2),
           "batch1_latency_ms": round(ms_b1, 3), "batch1_latency_graph_ms": ms_b1_graph,
           "gpu_launches_per_forward": launches,
           "how": "spcv_cu_model_forward: every activation device-resident; strict = bit-exact "
                  "with the reference run_network (tests/test_model_files.py)"}
    if dist.world == 1 and not args.no_cpu:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as orc  # CPU baseline leg: the reference executor itself

        ref = orc.Ref()
        xs = x[:2].cpu().numpy()
        ref.run_model(blob, xs[:1])
        t0 = time.perf_counter()
        ref.run_model(blob, xs)
        dt = (time.perf_counter() - t0) / xs.shape[0]
        out["reference_cpu"] = {"images_per_s": round(1.0 / dt, 2), "cores": 1, "kind": "reference",
                                "sample": "run_network (oracle/_ref, default ExecOptions) on 2 images, "
                                          "one thread (the reference executor is single-threaded)"}
    return out


def run_reference(args, layers, images):
    """--impl reference: the reference's own CPU spmm_into (oracle/_ref) on all
    host threads; rank 0 only under torchrun, other ranks exit without work."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    n_img = min(args.cpu_images or images, images)  # default: the full per-GPU workload
    sample = [make_layer_data(L, n_img, 1000 * (li + 1)) for li, L in enumerate(layers)]
    kind, flops, times = cpu_reference_run(sample, args.steps, args.warmup, threads)
    tot = sum(times)
    value = flops * len(times) / tot / 1e9  # flops = one step's sample
    line = {
        "impl": "reference", "metric": "SpMM effective GFLOP/s (2*nnz*N)", "value": round(value, 3),
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / len(times) * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded, BASELINE config shapes)",
        "config": {"workload": f"{args.config}: {WORKLOAD_DESC[args.config]}",
                   "images_per_gpu": images, "global_batch": images * world,
                   "sample_images_per_step": n_img},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
                         "sample": f"{n_img} image(s) x all {len(layers)} layers per step, "
                                   f"(layer,image) units over {threads} threads"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
