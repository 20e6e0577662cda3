#!/bin/bash
# Device time (median of 9, spin-gated events) of the layers most sensitive to
# per-tile overhead, each checked against the oracle: tools/layers_ab.sh [tag]
run() { python tools/prof_layer.py --config $1 --layer $2 --reps 9 --warmup 3 --check 2 ${3:+--images $3} 2>&1 | grep -E "median|Error|MISMATCH|check" | grep -v "OK" | sed "s/(prep.*slots=[0-9]*//; s/^/[${3:-full}] /"; }
run c3 c3_s70_b4,c3_s90_b4,c3_s95_b4,c3_s90_b2,c3_s90_b1,c3_s95_b1
run c2-b256 pw4,pw5,pw6,pw7,pw12,pw13
run c5 c5_s98
run c4 b7_project,b8_expand,b12_project,b15_expand,head
run c2-b256 pw4,pw7,pw13 32
