#!/bin/bash
# A/B timing of library variants (lib/variants/libspcv_cu_<name>.so) on single
# layers, each also checked bit-exact against the oracle on a few images.
#   tools/ab.sh "main v1 v2" "c3:c3_s90_b4,c3_s90_b1 c2-b256:pw7,pw13"  [extra env]
vars=$1; specs=$2
for v in $vars; do
  if [ "$v" = main ]; then lib=paper_1911_09723_b200/lib/libspcv_cu.so; else lib=paper_1911_09723_b200/lib/variants/libspcv_cu_$v.so; fi
  for spec in $specs; do
    cfg=${spec%%:*}; layers=${spec#*:}
    SPCV_CU_LIB=$lib timeout 600 python tools/prof_layer.py --config $cfg --layer $layers --reps 9 --warmup 3 --check ${CHECK:-2} 2>&1 \
      | grep -E "median|check|Error|error" | sed "s/^/[$v] /"
  done
done
