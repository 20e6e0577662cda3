#!/usr/bin/env python3
"""Annotate cuobjdump -sass output with the control bits of each instruction
(stall cycles, yield, read/write scoreboard, wait mask).

  cuobjdump -sass -fun NAME lib.so | python tools/sass_ctrl.py [--from ADDR --to ADDR]
"""
import re
import sys

lines = sys.stdin.read().splitlines()
args = sys.argv[1:]
lo = int(args[args.index("--from") + 1], 16) if "--from" in args else 0
hi = int(args[args.index("--to") + 1], 16) if "--to" in args else 1 << 40
pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(.*?);\s*/\* (0x[0-9a-f]{16}) \*/")
i = 0
total_stall = 0
while i < len(lines):
    m = pat.search(lines[i])
    if m and i + 1 < len(lines):
        m2 = re.search(r"/\* (0x[0-9a-f]{16}) \*/", lines[i + 1])
        if m2:
            addr = int(m.group(1), 16)
            lo64 = int(m.group(3), 16)
            hi64 = int(m2.group(1), 16)
            word = lo64 | (hi64 << 64)
            stall = (word >> 105) & 0xF
            yld = (word >> 109) & 1
            wbar = (word >> 110) & 7
            rbar = (word >> 113) & 7
            wait = (word >> 116) & 0x3F
            if lo <= addr <= hi:
                total_stall += stall
                print(f"{addr:05x} S{stall:2d} {'Y' if yld else ' '} w{wbar if wbar != 7 else '-'} "
                      f"r{rbar if rbar != 7 else '-'} m{wait:02x}  {m.group(2).strip()}")
            i += 2
            continue
    i += 1
print(f"sum of stall fields in range: {total_stall}", file=sys.stderr)
