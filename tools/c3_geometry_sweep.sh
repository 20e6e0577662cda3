#!/bin/bash
# CTA size x tail split on the c3 ablation layers (392 tiles over 148 SMs: 1.3 waves of 2 CTAs per SM)
for l in c3_s90_b4 c3_s70_b4 c3_s95_b4 c3_s90_b2 c3_s90_b1; do
for e in "" "SPCV_TAIL=2" "SPCV_TAIL=4" "SPCV_NWARPS=4" "SPCV_NWARPS=4 SPCV_TAIL=0" "SPCV_NWARPS=4 SPCV_TAIL=2" "SPCV_NWARPS=16" "SPCV_SPLIT=2"; do
env $e python tools/prof_layer.py --config c3 --layer $l --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
done; done
