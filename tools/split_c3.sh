#!/bin/bash
for sp in 0 1 2 4; do
  if [ $sp = 0 ]; then envs=""; else envs="SPCV_SPLIT=$sp"; fi
  env $envs python tools/prof_layer.py --config c3 --layer c3_s70_b4,c3_s90_b4,c3_s95_b4,c3_s90_b2,c3_s90_b1 --reps 7 2>&1 \
    | grep -E "median" | sed -E "s/.*\] //; s/^/[split=$sp] /; s/kernel=\S+ .*median/median/; s/GFLOP.*//"
  env $envs python tools/prof_layer.py --config c4 --layer b8_expand,b12_project,b15_expand,head --reps 7 2>&1 \
    | grep -E "median" | sed -E "s/.*\] //; s/^/[split=$sp] /; s/kernel=\S+ .*median/median/; s/GFLOP.*//"
done
