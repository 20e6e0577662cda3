#!/usr/bin/env python3
"""Summarise ncu reports (run here, no GPU needed).

  python tools/ncu_summary.py gpurun_out/r1_pw7.ncu-rep [...]        # key metrics
  python tools/ncu_summary.py --traffic profiles/traffic_latest.json name=rep ...
  python tools/ncu_summary.py --launches gpurun_out/r1_launches.csv  # per-launch list

The key metrics are the ones SURVEY.md §8d asks for: DRAM bytes, L2 hit rate,
L1/shared wavefronts (the gather roof), FMA pipe, issue, occupancy, stalls.
"""
import argparse
import csv
import json
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed (avg per SM)"),
    ("smsp__cycles_active.avg", "SMSP cycles active (avg)"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data-pipe wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg", "global-load wavefronts per SM"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared load bank conflicts"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % (active)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy % (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active % (active)"),
    ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active", "FMA-heavy pipe cycles % (active)"),
    ("smsp__inst_executed.sum", "warp instructions executed"),
    ("smsp__warps_eligible.avg.per_cycle_active", "eligible warps per cycle"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall: short scoreboard"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall: long scoreboard"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall: MIO throttle"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall: wait"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall: barrier"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    kname = rows[2][rows[0].index("Kernel Name")] if "Kernel Name" in rows[0] else "?"
    return kname, {n: (u, v) for n, u, v in zip(rows[0], rows[1], rows[2])}


def summary(rep):
    kname, d = raw(rep)
    lines = [f"report: {rep}", f"kernel: {kname}"]
    for k, label in KEYS:
        if k in d:
            lines.append(f"  {label:42s} {d[k][1]:>16s} {d[k][0]}")
    return "\n".join(lines)


def dram_bytes(rep):
    _, d = raw(rep)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        u, v = d[k]
        tot += float(v) * scale.get(u, 1)
    return tot


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    out = []
    for r in rows[1:]:
        x = dict(zip(h, r))
        out.append(f'{x["ID"]:>4s} {x["Kernel Name"][:48]:48s} grid {x["Grid Size"]:>16s} '
                   f'block {x["Block Size"]:>12s} {float(x["Metric Value"]) / 1e3:10.1f} us')
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="*")
    ap.add_argument("--traffic", default=None, help="write {name: dram bytes per launch} json")
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    if a.launches:
        print(launches(a.launches))
    elif a.traffic:
        t = {}
        for spec in a.reps:
            name, rep = spec.split("=", 1)
            t[name] = dram_bytes(rep)
        json.dump(t, open(a.traffic, "w"), indent=1)
        print(json.dumps(t, indent=1))
    else:
        for r in a.reps:
            print(summary(r))
            print()
