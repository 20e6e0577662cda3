#!/usr/bin/env python3
"""One bench step of a config between cudaProfilerStart/Stop, after warm-up
(and the first-call geometry autotuning), for
`ncu --profile-from-start off ...`: the captured launches are exactly the
step's layers, in order.

  ncu --profile-from-start off --clock-control none --csv \
      --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      python tools/step_profile.py [--config c2-b256] > step.csv
  python tools/step_profile.py --traffic step.csv [--config c2-b256] > profiles/traffic_latest.json
"""
import argparse
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def traffic(path, names):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    iM, iV, iID, iU = h.index("Metric Name"), h.index("Metric Value"), h.index("ID"), h.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = collections.OrderedDict()
    for r in rows:
        if r[iM] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[r[iID]] = per.get(r[iID], 0.0) + float(r[iV].replace(",", "")) * scale.get(r[iU], 1)
    vals = list(per.values())
    if len(vals) != len(names):
        raise SystemExit(f"{len(vals)} launches in {path}, expected {len(names)}")
    return dict(zip(names, vals))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2-b256")
    ap.add_argument("--images", type=int, default=None)
    ap.add_argument("--mode", choices=["strict", "fast"], default="strict")
    ap.add_argument("--traffic", default=None, help="ncu csv of this script -> {layer: DRAM bytes per launch}")
    args = ap.parse_args()
    from paper_1911_09723_b200.workloads import CONFIGS

    layers = CONFIGS[args.config]["layers"]()
    if args.traffic:
        print(json.dumps(traffic(args.traffic, [L.name for L in layers]), indent=1))
        return
    import torch

    import bench
    import paper_1911_09723_b200 as sp

    images = args.images or CONFIGS[args.config]["images"]
    data = bench.gen_data(layers, images, 0)
    dev_layers = bench.upload(sp, data, images, 0, args.mode)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        for _ in range(3):
            for (dw, a, b, o, fused, cfgk) in dev_layers:
                sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        for (dw, a, b, o, fused, cfgk) in dev_layers:
            sp.spmm_batched_into(dw, a, b, fused, o, cfgk, stream=stream)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
