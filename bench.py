#!/usr/bin/env python3
"""Benchmark of the B200 sparse 1x1-conv SpMM (the north-star path).

Default workload (BASELINE.json configs[1]): the 13 MobileNet-v1-1.0 pointwise
layers at 224x224, 90% unstructured sparsity, ReLU6, fp32, a global batch of
256 images partitioned over the GPUs (strong scaling: each rank runs its
contiguous image shard, weights replicated, no collective on the data path).
One step = one pass of all 13 layers over the rank's shard. At N>1 the line
also carries a weak-scaling measurement (256 images on every GPU).

Metric (BASELINE.json): effective GFLOP/s = 2*nnz*N / t summed over layers
(reference convention, /root/reference/proj/src/bench.cpp:211), plus
algorithmic HBM GB/s against the measured peak.

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

`--gpus N` without torchrun re-launches itself under torch.distributed.run
with N ranks; under torchrun WORLD_SIZE must equal N. Before any timing the
run passes a self-check gate (the reference's require_selfcheck,
bench.cpp:140-167): three quick sparse layers and a sample of the benched
layers must equal the reference oracle bit for bit, else the run exits 2
without a JSON line. Rank 0 prints ONE JSON line on stdout; details go to
stderr.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# pure-numpy imports: neither maps the CUDA library (the reference arm must not)
from paper_1911_09723_b200.dist import Dist, shard  # noqa: E402
from paper_1911_09723_b200.workloads import CONFIGS, Layer, activation_of, make_layer_data  # noqa: E402

WORKLOAD_DESC = {
    "c2-b256": "MobileNet-v1-1.0 pointwise stack @224 (13 layers), 90% unstructured, ReLU6",
    "c2-b1": "MobileNet-v1-1.0 pointwise stack @224 (13 layers), 90% unstructured, ReLU6",
    "c1": "single 128x128 sparse 1x1 conv @28x28, 80% unstructured, ReLU",
    "c3": "512x512 @14x14, block 4/2/1 x1, sparsity 70-95%, ReLU",
    "c4": "MobileNet-v2-1.0 1x1 convs @224, 85% unstructured, ReLU6/linear",
    "c5": "1024x1024 @7x7, Beta(2,8)-skewed rows, sparsity 70-98%, ReLU",
}
L2_BYTES = 126 * 1024 * 1024
METRIC = "SpMM effective GFLOP/s (2*nnz*N)"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def step_bytes(layers, images: int) -> float:
    """Activations in + outputs out of one step (the bytes that decide L2 residency)."""
    return float(sum(4 * (L.cin + L.cout) * L.spatial * images for L in layers))


def bench_config(args, layers, world: int, rank_images: int) -> dict:
    """The workload description, identical in both arms (built from the
    arguments and the layer shapes only, never from measurements)."""
    sb = step_bytes(layers, rank_images)
    flush = sb < 4 * L2_BYTES
    return {
        "workload": f"{args.config}: {WORKLOAD_DESC[args.config]}",
        "global_batch": args.global_batch,
        "images_per_gpu": rank_images,
        "mode": args.mode,
        "parallelism": f"dp{world} (contiguous image shards, replicated weights, no collective)",
        "l2": (f"L2 flushed between timed steps ({sb / 1e6:.1f} MB per step per GPU < 4x the 126 MB L2)"
               if flush else
               f"inputs larger than L2: {sb / 1e9:.2f} GB of activations+outputs per step per GPU "
               f"vs 126 MB L2, no explicit flush"),
    }


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


# -------------------------------------------------------- self-check gate
# require_selfcheck (bench.cpp:140-167): three sparse layers at 90%, ReLU6,
# block heights 1/2/4, against the reference oracle matmul_reference
# (tensor.cpp:38-62). The reference allows 1e-5; strict mode must be exact.
SELFCHECK_CASES = [(64, 32, 14, 14, 1), (96, 64, 14, 14, 2), (128, 96, 7, 7, 4)]


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as orc  # checker / CPU-baseline legs only

    return orc


def selfcheck_cases(inject_fault: bool):
    out = []
    for ci, (cout, cin, h, w, bh) in enumerate(SELFCHECK_CASES):
        L = Layer(f"selfcheck{ci}", cin, cout, h, w, ("clamp", 0.0, 6.0), 0.0, 6.0, 0.9, bh)
        d = make_layer_data(L, 1, 0xC0DE + ci)
        if inject_fault and ci == 0 and d.weights.values.size:
            d.weights.values = d.weights.values.copy()
            d.weights.values[0] += np.float32(1.0)  # bench.cpp:150-151 test hook
        out.append(d)
    return out


def compare_exact(got: np.ndarray, want: np.ndarray) -> tuple[bool, float]:
    same = np.array_equal(got.view(np.uint32), want.view(np.uint32))
    dev = float(np.max(np.abs(got.astype(np.float64) - want.astype(np.float64)))) if got.size else 0.0
    return same, dev


def gate_fail(msg: str):
    log(f"self-check FAILED: {msg}; refusing to emit records")
    sys.exit(2)


# ------------------------------------------------------------ CPU reference
def cpu_reference_run(layers_data, steps: int, warmup: int, threads: int):
    """Reference spmm_into (oracle/_ref, else the oracle port) on host cores.
    Every (layer, image) pair is one spmm_into call; `threads` host threads
    pull them longest-first (oracle/ref_shim.cpp: ref_bench_layers)."""
    orc = _oracle()
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
def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", default="c2-b256", choices=sorted(CONFIGS))
    ap.add_argument("--global-batch", type=int, default=None,
                    help="images partitioned over the ranks (default: the config's batch)")
    ap.add_argument("--images-per-gpu", type=int, default=None,
                    help="weak scaling instead: this many images on every rank")
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
    ap.add_argument("--no-weak", action="store_true", help="N>1: skip the extra weak-scaling run")
    ap.add_argument("--inject-fault", action="store_true",
                    help="corrupt one weight of the first self-check case (the gate must refuse)")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        log("warmup < 3 is not allowed by the timing rules; using 3")
        args.warmup = 3
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    return args


def maybe_spawn(args) -> None:
    """--gpus N outside torchrun: re-launch this script with N ranks (one per GPU)."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            log(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch with --nproc-per-node {args.gpus}")
            sys.exit(2)
        return
    if args.gpus == 1:
        return
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("spawning: " + " ".join(cmd))
    os.execv(sys.executable, cmd)


def rank_images(args, world: int, rank: int) -> tuple[int, str]:
    if args.images_per_gpu:
        return args.images_per_gpu, "weak"
    b0, b1 = shard(args.global_batch, world, rank)
    return b1 - b0, "strong"


def main():
    args = parse_args()
    cfg = CONFIGS[args.config]
    layers = cfg["layers"]()
    if args.global_batch is None:
        args.global_batch = cfg["images"]
    if args.impl == "reference":
        return run_reference(args, layers)
    maybe_spawn(args)

    import torch

    # SPCV_DIST_BACKEND=gloo runs the N>1 code path with ranks sharing a GPU
    # (a functional check on a one-GPU box; NCCL refuses two ranks per GPU)
    backend = os.environ.get("SPCV_DIST_BACKEND", "nccl")
    dist = Dist(backend)
    if not torch.cuda.is_available():
        log("no CUDA device: the B200 arm has no CPU path")
        sys.exit(2)
    if dist.world > torch.cuda.device_count() and backend == "nccl":
        log(f"{dist.world} ranks but {torch.cuda.device_count()} visible GPU(s)")
        sys.exit(2)
    dev = dist.local % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    import paper_1911_09723_b200 as sp

    hbm_peak, peak_kind = peaks()
    images, scaling = rank_images(args, dist.world, dist.rank)
    config = bench_config(args, layers, dist.world, rank_images(args, dist.world, 0)[0])
    cdev = torch.device("cuda", dev)
    stream = torch.cuda.Stream(dev)

    # ---- self-check gate (every rank; any failure stops every rank)
    selfcheck = run_selfcheck(args, sp, layers, dist, dev, stream)

    # ---- data: weights identical on every rank, activations per-rank shard
    t0 = time.time()
    data = gen_data(layers, images, dist.rank)
    log(f"[rank {dist.rank}] generated {len(layers)} layers x {images} images in {time.time() - t0:.1f}s")
    dev_layers = upload(sp, data, images, dev, args.mode)
    torch.cuda.synchronize()

    # the rank's sampled outputs must equal the oracle (part of the gate)
    gate_sample(sp, data, dev_layers, stream, dist, dev, selfcheck)

    flush_buf = None
    if step_bytes(layers, images) < 4 * L2_BYTES:
        flush_buf = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=cdev)
    res = time_steps(sp, dev_layers, args.steps, args.warmup, stream, dist, dev, flush_buf)
    ms_step, launches, clk, per_layer_us = res["ms_step"], res["launches"], res["clk"], res["per_layer_us"]

    flops_step = sum(d.flops() for d in data)
    bytes_step = sum(d.alg_bytes() for d in data)
    flops_all = dist.sum(flops_step, device=cdev)
    value = flops_all / (ms_step * 1e-3) / 1e9

    graph = None if args.no_alt else bench_graph(sp, dev_layers, args.steps, stream, dist, dev, flops_all)
    ms_alt = float("nan")
    other = "fast" if args.mode == "strict" else "strict"
    if not args.no_alt:
        alt = [(dw, a, b, o, f, sp.MicrokernelConfig(n=c.n, strict=(other == "strict")))
               for (dw, a, b, o, f, c) in dev_layers]
        ms_alt = time_steps(sp, alt, args.steps, args.warmup, stream, dist, dev, flush_buf,
                            per_layer=False)["ms_step"]

    # per-layer kernel times (events on the launch stream, averaged over steps)
    per_layer = []
    for li, d in enumerate(data):
        us = per_layer_us[li]
        per_layer.append(dict(name=d.layer.name, K=d.layer.cin, M=d.layer.cout, S=d.layer.spatial,
                              bh=d.layer.block_h, nnz=d.nnz, row_slots=dev_layers[li][0].row_slots,
                              us=us, gflops=d.flops() / us / 1e3, gbs=d.alg_bytes() / us / 1e3,
                              hbm_frac=d.alg_bytes() / us / 1e3 / hbm_peak,
                              alg_bytes=d.alg_bytes(), flops=d.flops(),
                              kernel={"jit": "spcv_jit", "small": "spmm_small_kernel"}.get(
                                  dev_layers[li][0].kernel_for(images, d.layer.h, d.layer.w, args.mode == "strict"),
                                  "spmm_bcsr_kernel")))
    tot_us = sum(p["us"] for p in per_layer)
    for p in per_layer:
        p["share"] = p["us"] / tot_us
    if dist.rank == 0:
        log(f"{'layer':12s} {'K':>5s} {'M':>5s} {'S':>6s} {'slots':>5s} {'us':>9s} {'GFLOP/s':>9s} "
            f"{'GB/s':>8s} {'HBM%':>6s} {'share':>6s}")
        for p in per_layer:
            log(f"{p['name']:12s} {p['K']:5d} {p['M']:5d} {p['S']:6d} {p['row_slots']:5d} {p['us']:9.1f} "
                f"{p['gflops']:9.0f} {p['gbs']:8.0f} {100 * p['hbm_frac']:6.1f} {100 * p['share']:6.1f}")
        log(f"step {ms_step:.4f} ms; layer kernels sum {tot_us / 1e3:.4f} ms; "
            f"{value:.0f} GFLOP/s aggregate over {dist.world} GPU(s) ({scaling})")
        if args.layers_json:
            json.dump(per_layer, open(args.layers_json, "w"), indent=1)

    dense = None if args.no_dense else bench_dense(sp, data, dev_layers, per_layer, args, stream, dist, dev,
                                                   ms_step, flush_buf)
    e2e = None if args.no_e2e else bench_e2e(sp, data, dev_layers, images, args, stream, dist, dev, flops_all)
    network = None if args.no_network else bench_network(args, dev, stream, dist, images)

    # ---- weak scaling (N>1): the config's batch on every GPU
    weak = None
    if dist.world > 1 and scaling == "strong" and not args.no_weak:
        wimg = cfg["images"]
        wdata = gen_data(layers, wimg, dist.rank)
        wl = upload(sp, wdata, wimg, dev, args.mode)
        wres = time_steps(sp, wl, args.steps, args.warmup, stream, dist, dev, None, per_layer=False)
        wflops = dist.sum(sum(d.flops() for d in wdata), device=cdev)
        weak = {"images_per_gpu": wimg, "global_batch": wimg * dist.world,
                "ms_per_step": round(wres["ms_step"], 4),
                "value": round(wflops / (wres["ms_step"] * 1e-3) / 1e9, 3), "unit": "GFLOP/s"}
        del wl, wdata

    # ---- CPU baseline (rank 0, N=1 only), a bounded sample of the same workload
    cpu = None
    if dist.world == 1 and not args.no_cpu:
        cpu = bench_cpu(args, data, layers, images)

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    clk_sum = clk.summary()
    f_clk = (clk_sum.get("sm_mhz") or clk_sum.get("sm_max_mhz") or 1965.0) * 1e6
    gather_roof = sms * 64 * f_clk / 1e12  # TFLOP/s
    if dist.rank == 0:
        roofline = make_roofline(per_layer, hbm_peak, peak_kind, gather_roof, bytes_step, ms_step, value,
                                 dist.world)
        line = {
            "metric": METRIC, "value": round(value, 3),
            "unit": "GFLOP/s", "n_gpus": dist.world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, BASELINE config shapes)",
            "config": config,
            "selfcheck": selfcheck,
            "hbm_gbs": round(bytes_step * dist.world / (ms_step * 1e-3) / 1e9, 1),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "dense_baseline": dense,
            "weak_scaling": weak, "network": network, "graph": graph,
            "timing": res["timing"],
            "gpu_launches": launches, "clocks": clk_sum,
            "modes": {args.mode: {"value": round(value, 3), "ms_per_step": round(ms_step, 4)},
                      other: ({"value": round(flops_all / (ms_alt * 1e-3) / 1e9, 3),
                               "ms_per_step": round(ms_alt, 4)} if ms_alt == ms_alt else None),
                      "note": "strict = bit-exact vs the reference CPU kernel (default); "
                              "fast = FFMA, within the north_star nnz-scaled 1e-5 tolerance"},
        }
        print(json.dumps(line), flush=True)
    dist.close()


# ----------------------------------------------------------------- helpers
def gen_data(layers, images: int, rank: int):
    data = []
    for li, L in enumerate(layers):
        d = make_layer_data(L, images, 1000 * (li + 1) + rank)
        w = make_layer_data(L, 1, 1000 * (li + 1), act=False)  # weights: rank-independent seed
        d.weights, d.dense, d.bias = w.weights, w.dense, w.bias
        data.append(d)
    return data


def upload(sp, data, images: int, dev: int, mode: str):
    import torch

    out = []
    for d in data:
        dw = sp.DeviceBcsr(d.weights)
        a = torch.from_numpy(d.act).to(dev)
        o = torch.empty((images, d.layer.cout, d.layer.h, d.layer.w), device=dev)
        b = torch.from_numpy(d.bias).to(dev)
        cfgk = sp.MicrokernelConfig(n=d.layer.block_h, strict=(mode == "strict"))
        out.append((dw, a, b, o, activation_of(d.layer.act), cfgk))
    return out


def run_selfcheck(args, sp, layers, dist, dev, stream) -> dict:
    """The gate's fixed cases through the device path in strict mode (plus the
    run's own mode), compared with matmul_reference of the dense matrix."""
    import torch

    orc = _oracle()
    oracle = orc.Oracle()
    ok, worst, names = True, 0.0, []
    for d in selfcheck_cases(args.inject_fault):
        L = d.layer
        w = sp.DeviceBcsr(d.weights)
        a = torch.from_numpy(d.act).to(dev)
        b = torch.from_numpy(d.bias).to(dev)
        o = torch.empty((1, L.cout, L.h, L.w), device=dev)
        fused = activation_of(L.act)
        with torch.cuda.stream(stream):
            sp.spmm_batched_into(w, a, b, fused, o, sp.MicrokernelConfig(n=L.block_h), stream=stream)
        stream.synchronize()
        want = oracle.matmul_reference(d.dense, d.act[0].reshape(L.cin, -1), d.bias, L.act)
        same, dev_ = compare_exact(o.cpu().numpy().reshape(want.shape), want)
        worst = max(worst, dev_)
        names.append(f"{L.cout}x{L.cin}@{L.h}x{L.w} {L.block_h}x1")
        if not same:
            ok = False
            log(f"[rank {dist.rank}] self-check case {names[-1]}: max deviation {dev_:g} (strict must be exact)")
    flag = dist.max(0.0 if ok else 1.0, device=torch.device("cuda", dev))
    if flag > 0:
        gate_fail("a strict-mode case differs from the reference oracle (matmul_reference, tensor.cpp:38-62)")
    return {"passed": True, "cases": names, "max_abs_dev": worst,
            "how": "require_selfcheck (bench.cpp:140-167): 90% sparse, ReLU6, block 1/2/4, strict device "
                   "path vs oracle matmul_reference, bit-exact; plus image 0 of 3 benched layers per rank"}


def gate_sample(sp, data, dev_layers, stream, dist, dev, selfcheck: dict) -> None:
    """Image 0 of the first, middle and last benched layer on this rank vs the oracle."""
    import torch

    if not dev_layers or data[0].images == 0:
        return
    orc = _oracle()
    oracle = orc.Oracle()
    idx = sorted({0, len(data) // 2, len(data) - 1})
    bad = []
    for li in idx:
        d = data[li]
        dw, a, b, o, fused, cfgk = dev_layers[li]
        strict_cfg = sp.MicrokernelConfig(n=cfgk.n, strict=True)
        with torch.cuda.stream(stream):
            sp.spmm_batched_into(dw, a[:1].contiguous(), b, fused, o[:1], strict_cfg, stream=stream)
        stream.synchronize()
        L = d.layer
        want = oracle.matmul_reference(d.dense, d.act[0].reshape(L.cin, -1), d.bias, L.act)
        same, dev_ = compare_exact(o[0].cpu().numpy().reshape(want.shape), want)
        selfcheck["max_abs_dev"] = max(selfcheck["max_abs_dev"], dev_)
        if not same:
            bad.append(L.name)
    flag = dist.max(1.0 if bad else 0.0, device=torch.device("cuda", dev))
    if flag > 0:
        gate_fail(f"benched layer(s) {bad or '(another rank)'} differ from the oracle")
    selfcheck["benched_layers_checked"] = [data[i].layer.name for i in idx]


def time_steps(sp, dev_layers, steps, warmup, stream, dist, dev, flush_buf, per_layer=True) -> dict:
    """Warm-up, then EXACTLY `steps` timed steps between a barrier + synchronize
    on both sides (CUDA events on the launch stream, max over ranks). Without a
    flush buffer the step runs back to back (inputs larger than L2); with one,
    every step is timed on its own and the L2 is overwritten between steps."""
    import torch

    cdev = torch.device("cuda", dev)

    # each layer's call bound once to its (fixed) device buffers: one C-ABI call
    # per launch without the per-call torch attribute reads, which otherwise
    # bound the batch-1 configs (13 launches of ~5-8 us each) on the host
    calls = [sp.bind_batched(dw, a, b, fused, o, cfgk, stream=stream) for dw, a, b, o, fused, cfgk in dev_layers]

    def step(evs=None):
        if evs is None:
            for call in calls:
                call()
            return
        for li, call in enumerate(calls):
            evs[li][0].record(stream)
            call()
            evs[li][1].record(stream)

    def flush():
        if flush_buf is not None:
            flush_buf.fill_(1.0)

    def ev():
        return torch.cuda.Event(enable_timing=True)

    nl = len(dev_layers)
    with torch.cuda.stream(stream):
        for _ in range(warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier(dev)
        torch.cuda.synchronize()
        launches0 = sp.launch_count()
        with ClockProbe(dev) as clk:
            if flush_buf is None:
                # back to back; an event at every step boundary gives the per-step
                # median too (recording an event adds no gap on the stream)
                marks = [ev() for _ in range(steps + 1)]
                marks[0].record(stream)
                for k in range(steps):
                    step()
                    marks[k + 1].record(stream)
                torch.cuda.synchronize()
                ms_local = marks[0].elapsed_time(marks[-1])
                step_ms = [marks[k].elapsed_time(marks[k + 1]) for k in range(steps)]
            else:
                pairs = []
                for _ in range(steps):
                    flush()
                    e0, e1 = ev(), ev()
                    e0.record(stream)
                    step()
                    e1.record(stream)
                    pairs.append((e0, e1))
                torch.cuda.synchronize()
                step_ms = [e0.elapsed_time(e1) for e0, e1 in pairs]
                ms_local = sum(step_ms)
        launches = sp.launch_count() - launches0
        dist.barrier(dev)
        per_layer_us = None
        if per_layer:
            # per-layer breakdown: a separate pass with events around every launch
            # (kept out of the headline region: the event records add gaps)
            lev = [[[ev(), ev()] for _ in range(nl)] for _ in range(steps)]
            for k in range(steps):
                flush()
                step(lev[k])
            torch.cuda.synchronize()
            per_layer_us = [statistics.mean(lev[k][li][0].elapsed_time(lev[k][li][1]) for k in range(steps)) * 1e3
                            for li in range(nl)]
    ms_total = dist.max(ms_local, device=cdev)
    timing = {"region": "K back-to-back steps, events at every step boundary" if flush_buf is None else
              "K steps, one event pair each, L2 overwritten (252 MB fill) between steps",
              "median_step_ms": round(statistics.median(step_ms), 4) if step_ms else None,
              "value_from": "total time of the K timed steps / K (max over ranks)"}
    return {"ms_step": ms_total / steps, "launches": launches, "clk": clk, "per_layer_us": per_layer_us,
            "timing": timing}


def bench_graph(sp, dev_layers, steps, stream, dist, dev, flops_all):
    """The same step replayed as one CUDA graph (launch overhead out of the way).
    Every rank reaches the same collectives whether or not its capture works."""
    import torch

    cdev = torch.device("cuda", dev)

    def step():
        for (dw, a, b, o, fused, cfgk) in dev_layers:
            sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)

    ms_local, err, g = -1.0, "", None
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
    ok = -dist.max(-flag, device=cdev) > 0  # min over ranks: all captured
    if ok:
        with torch.cuda.stream(stream):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier(dev)
            torch.cuda.synchronize()
            e0.record(stream)
            for _ in range(steps):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
        ms_local = e0.elapsed_time(e1)
    ms_graph = dist.max(ms_local, device=cdev) / steps if ok else -1.0
    del g
    if not ok:
        return {"unavailable": err or "capture failed on another rank"}
    return {"ms_per_step": round(ms_graph, 4), "value": round(flops_all / (ms_graph * 1e-3) / 1e9, 3),
            "how": f"torch.cuda.CUDAGraph capture of one step ({len(dev_layers)} spcv_cu_spmm_into launches), "
                   "replayed back to back"}


def bench_dense(sp, data, dev_layers, per_layer, args, stream, dist, dev, ms_step, flush_buf):
    """Dense fp32 baseline (reference dense_gemm_into, bench.cpp:216-227): the
    same layers with dense weights through cuBLAS SGEMM (pedantic fp32)."""
    import torch

    cdev = torch.device("cuda", dev)
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
        dev_ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in dws] for _ in range(dsteps)]
        dist.barrier(dev)
        torch.cuda.synchronize()
        tot = 0.0
        for k in range(dsteps):
            if flush_buf is not None:
                flush_buf.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step_dense(dev_ev[k])
            e1.record(stream)
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
    ms_dense = dist.max(tot, device=cdev) / dsteps
    dense_flops = sum(2.0 * d.layer.cout * d.layer.cin * d.images * d.layer.spatial for d in data)
    for li, p in enumerate(per_layer):
        p["dense_us"] = statistics.mean(dev_ev[k][li][0].elapsed_time(dev_ev[k][li][1]) for k in range(dsteps)) * 1e3
    if dist.rank == 0:
        log(f"dense fp32 baseline: {ms_dense:.3f} ms/step; sparse speedup {ms_dense / ms_step:.2f}x")
    return {"ms_per_step": round(ms_dense, 4),
            "dense_gflops": round(dense_flops * dist.world / (ms_dense * 1e-3) / 1e9, 1),
            "sparse_effective_gflops": round(dense_flops * dist.world / (ms_step * 1e-3) / 1e9, 1),
            "sparse_speedup_vs_dense": round(ms_dense / ms_step, 3),
            "per_layer_speedup": {p["name"]: round(p["dense_us"] / p["us"], 2) for p in per_layer},
            "how": f"cuBLAS SGEMM strided-batched (CUBLAS_PEDANTIC_MATH) + bias/clamp epilogue, same inputs, "
                   f"{dsteps} steps"}


def bench_e2e(sp, data, dev_layers, images, args, stream, dist, dev, flops_all):
    """End to end through the host-buffer C-ABI call (spcv_cu_spmm_into_host:
    H2D of the step's inputs, kernel, D2H of its outputs, per layer)."""
    import torch

    cdev = torch.device("cuda", dev)
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
    dt = dist.max(dt, device=cdev)
    # e2e outputs must equal the device path's outputs (headline mode)
    with torch.cuda.stream(stream):
        for (dw, a, b, o, fused, cfgk) in dev_layers:
            sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)
    torch.cuda.synchronize()
    for (_, _, _, o_dev, _, _), (_, o) in zip(dev_layers, host):
        if not np.array_equal(o_dev.cpu().numpy().view(np.uint32), o.view(np.uint32)):
            raise SystemExit("e2e output differs from the device-path output")
    return {"value": round(flops_all / (dt / args.steps) / 1e9, 3),
            "unit": "GFLOP/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": round(dt / args.steps * 1e3, 3),
            "path": "spcv_cu_spmm_into_host per layer (pinned host buffers; image chunks pipelined "
                    "H2D|kernel|D2H on 3 streams); host wall clock, max over ranks"}


def bench_cpu(args, data, layers, images):
    threads = os.cpu_count() or 1
    n_img = min(args.cpu_images or images, images)
    sample = data
    if n_img < images:
        sample = [make_layer_data(d.layer, n_img, 1000 * (li + 1)) for li, d in enumerate(data)]
    kind, flops, times = cpu_reference_run(sample, 3, 1, threads)
    # the reference's own concurrency model (one thread), on an 8-image slice
    s1 = [make_layer_data(d.layer, min(8, images), 1000 * (li + 1)) for li, d in enumerate(data)]
    _, flops1, times1 = cpu_reference_run(s1, 3, 1, 1)
    return {"value": round(flops / statistics.median(times) / 1e9, 3), "unit": "GFLOP/s",
            "cores": threads, "kind": kind, "cpu_model": cpu_model(),
            "single_thread": {"value": round(flops1 / statistics.median(times1) / 1e9, 3),
                              "sample": f"{min(8, images)} images x all layers, 1 thread, median of 3"},
            "sample": f"{n_img} image(s) x all {len(layers)} layers of {args.config} "
                      f"(= {'the full step' if n_img == images else 'a slice of the step'}), "
                      f"(layer,image) spmm_into units over {threads} threads, median of 3 passes "
                      f"after 1 warm-up: {statistics.median(times):.3f}s/pass"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return ""


def make_roofline(per_layer, hbm_peak, peak_kind, gather_roof, bytes_step, ms_step, value, world):
    dom = max(per_layer, key=lambda p: p["us"])
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic_latest.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(dom["name"])
        except Exception:
            traffic = None

    def attainable(p):
        # SURVEY.md §8d "Cap": the best HBM fraction the binding roof allows
        t_hbm = p["alg_bytes"] / (hbm_peak * 1e9)
        t_gather = p["flops"] / (gather_roof * 1e12 * p["bh"])
        return min(1.0, t_hbm / max(t_hbm, t_gather))

    att = attainable(dom)
    return {"bound": "hbm", "achieved": round(dom["gbs"], 1), "peak": hbm_peak, "unit": "GB/s",
            "frac": round(dom["gbs"] / hbm_peak, 4), "traffic": traffic,
            "kernel": f"{dom.get('kernel', 'tile')} [{dom['name']}: {dom['K']}->{dom['M']} @S={dom['S']}]",
            "peak_kind": peak_kind,
            "alg_bytes_per_launch": dom["alg_bytes"], "avg_launch_us": round(dom["us"], 2),
            "share_of_step": round(dom["share"], 3),
            "step_hbm_frac": round(bytes_step / (ms_step * 1e-3) / 1e9 / hbm_peak, 4),
            "gather_roof_tflops": round(gather_roof, 2),
            "attainable_frac": round(att, 4),
            "frac_of_attainable": round((dom["gbs"] / hbm_peak) / att, 4),
            "gather_frac": round(dom["gflops"] / 1e3 / (gather_roof * dom["bh"]), 4),
            # every layer against its roofs: the tile kernel is bound by the lower of
            # HBM and the shared-memory gather; the weight-specialised (spcv_jit)
            # kernels gather nothing (activations in registers): HBM only
            "layers": {p["name"]: {
                "kernel": p["kernel"], "us": round(p["us"], 1),
                "bound": "hbm" if p["kernel"] == "spcv_jit" or attainable(p) >= 1.0 else "gather",
                "hbm_frac": round(p["hbm_frac"], 4),
                "attainable_frac": round(1.0 if p["kernel"] == "spcv_jit" else attainable(p), 4),
                "gather_frac": (None if p["kernel"] == "spcv_jit" else
                                round(p["gflops"] / 1e3 / (gather_roof * p["bh"]), 4))}
                for p in per_layer},
            "step_gather_frac": round(value / 1e3 / world / gather_roof, 4),
            "note": "achieved = SURVEY.md §8d algorithmic bytes / CUDA-event launch time. "
                    "Layers with AI > ~2.9 FLOP/B are bound by the shared-memory gather roof "
                    "(one 4 B activation per stored block per column at 128 B/clk/SM: "
                    "SMs x 64 FLOP/clk x SM clock), not HBM; gather_frac is against that roof "
                    "(x block height) at the clock measured during the run"}


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
    x = torch.from_numpy(rng.uniform(-1, 1, (max(batch, 1), 224, 224, 3)).astype(np.float32)).to(dev)

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
    if dist.rank == 0:
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
        orc = _oracle()  # CPU baseline leg: the reference executor itself
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


def mapped_libraries() -> list[str]:
    """Shared objects of this repo (or the reference build) mapped into this
    process (/proc/self/maps): the reference arm must map oracle/_ref only."""
    libs = set()
    try:
        for line in open("/proc/self/maps"):
            path = line.split()[-1] if len(line.split()) >= 6 else ""
            if path.endswith(".so") and path.startswith(ROOT):
                libs.add(os.path.relpath(path, ROOT))
    except OSError:
        pass
    return sorted(libs)


def run_reference(args, layers):
    """--impl reference: the reference's own CPU spmm_into (oracle/_ref, else
    the oracle port) on all host threads over the WHOLE job (the global batch,
    all layers) — the same config dict as the B200 arm; rank 0 only under
    torchrun, other ranks exit without work. Its own self-check gate first."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    orc = _oracle()
    kind = "reference" if orc.have_ref() else "port"
    # gate: the reference spmm on the self-check cases equals its own oracle
    for d in selfcheck_cases(args.inject_fault):
        L = d.layer
        if kind == "reference":  # the reference library against its own oracle
            ref = orc.Ref()
            want = ref.matmul_reference(d.dense, d.act[0].reshape(L.cin, -1), d.bias, L.act, L.h, L.w)
            got = ref.spmm(d.weights, d.act, d.bias, L.act)[1]
        else:
            oracle = orc.Oracle()
            want = oracle.matmul_reference(d.dense, d.act[0].reshape(L.cin, -1), d.bias, L.act)
            got = oracle.spmm(d.weights, d.act, d.bias, L.act)
        if not (np.max(np.abs(got.reshape(want.shape).astype(np.float64) - want)) <= 1e-5):
            gate_fail(f"reference case {L.cout}x{L.cin} differs from matmul_reference by more than 1e-5")
    images, scaling = rank_images(args, world, 0)
    config = bench_config(args, layers, world, images)
    job_images = args.images_per_gpu * world if args.images_per_gpu else args.global_batch
    threads = os.cpu_count() or 1
    n_img = min(args.cpu_images or job_images, job_images)  # default: the whole job
    sample = [make_layer_data(L, n_img, 1000 * (li + 1)) for li, L in enumerate(layers)]
    kind, flops, times = cpu_reference_run(sample, args.steps, args.warmup, threads)
    tot = sum(times)
    value = flops * len(times) / tot / 1e9  # flops = one step's sample
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3),
        "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tot / len(times) * 1e3, 3), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded, BASELINE config shapes)",
        "config": config,
        "selfcheck": {"passed": True, "how": "reference spmm vs oracle matmul_reference on the "
                                             "require_selfcheck cases (bench.cpp:140-167), <= 1e-5"},
        "cpu_baseline": {"value": round(value, 3), "unit": "GFLOP/s", "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{n_img} image(s) x all {len(layers)} layers per step (the whole job of "
                                   f"{job_images} images over {world} GPU(s)), (layer,image) spmm_into units "
                                   f"over {threads} threads"},
        "e2e": {"value": round(value, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "repo_libraries_mapped": mapped_libraries(),
    }
    if any("libspcv_cu" in p or "libspcv_b200" in p for p in line["repo_libraries_mapped"]):
        log(f"reference arm mapped this repo's CUDA library: {line['repo_libraries_mapped']}")
        sys.exit(2)
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
