#!/usr/bin/env python3
"""Per-launch table from an ncu --csv metrics run (duration, DRAM bytes, issue).

  python tools/launch_table.py gpurun_out/net_launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h, rows = rows[0], rows[1:]
    iN, iM, iV, iID = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    d = collections.OrderedDict()
    for r in rows:
        d.setdefault(r[iID], {"name": r[iN][:56]})[r[iM]] = float(r[iV].replace(",", ""))
    tot = 0.0
    for k, v in d.items():
        t = v["gpu__time_duration.sum"] / 1e3
        tot += t
        mb = (v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)) / 1e6
        iss = v.get("smsp__issue_active.avg.pct_of_peak_sustained_active", float("nan"))
        print(f"{k:>4} {v['name']:56s} {t:8.1f} us {mb:8.1f} MB {mb / t:6.2f} TB/s issue {iss:3.0f}%")
    print(f"total {tot:.1f} us over {len(d)} launches")


if __name__ == "__main__":
    main(sys.argv[1])
