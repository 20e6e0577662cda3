#!/bin/bash
# Device time of the unaligned-layout (H*W % 4 != 0) layers, each checked against the oracle.
run() { python tools/prof_layer.py --config $1 --layer $2 --reps 9 --warmup 3 --check 2 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//"; }
run c2-b256 pw12,pw13
run c5 c5_s98,c5_s95,c5_s90,c5_s80,c5_s70
run c4 b14_project,b15_expand,b15_project,b17_project,head
