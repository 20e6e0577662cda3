#!/bin/bash
# Row split (CTAs per tile) sweep on mid-size calls: tools/split_ab.sh IMAGES LAYERS
img=$1; layers=$2
for sp in 0 1 2 4 8; do
  if [ $sp = 0 ]; then envs=""; else envs="SPCV_SPLIT=$sp"; fi
  env $envs python tools/prof_layer.py --config c2-b256 --layer $layers --images $img --reps 7 2>&1 \
    | grep -E "median" | sed -E "s/.*\] //; s/^/[img=$img split=$sp] /; s/kernel=\S+ .*median/median/; s/GFLOP.*//"
done
