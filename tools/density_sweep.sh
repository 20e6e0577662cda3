#!/bin/bash
# Steady state of the tile kernel without a tail: 2960 images of 4x4 = 1480 tiles of 32 columns = 10 per
# SM exactly; 512x512 matrices at several densities and block heights (profiles/r2_notes.md, r2f).
for bh in ${BHS:-4 1}; do for s in ${SPARS:-0.0 0.7 0.9}; do
python tools/prof_layer.py --adhoc 512,512,4,4,$s,$bh,2960 --reps 5 --warmup 2 --check 1 2>&1 | grep -E "median|Error" | sed "s/^/[bh=$bh s=$s] /; s/(prep.*slots=[0-9]*//"
done; done
