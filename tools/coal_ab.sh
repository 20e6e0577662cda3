#!/bin/bash
# Scattered vs coalesced epilogue on the unaligned (H*W = 49) layers: SPCV_COAL=0 / 2 (1 = autotuned).
for c in 0 2 1; do
  for spec in "c2-b256:pw12,pw13" "c5:c5_s98,c5_s95,c5_s90,c5_s70" "c4:b14_project,b15_expand,b15_project,b17_project,head"; do
    cfg=${spec%%:*}; layers=${spec#*:}
    SPCV_COAL=$c python tools/prof_layer.py --config $cfg --layer $layers --reps 9 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[coal=$c] /"
  done
done
