#!/bin/bash
# ncu --set full of single layers (one launch each, after warm-up and the
# first-call tail autotuning). Run on the GPU box:
#   tools/ncu_layers.sh TAG config:layer [config:layer ...]
# Leaves gpurun_out/TAG_<layer>.{summary.txt,raw.csv,details.txt,sass.csv}; the
# .ncu-rep itself is deleted (too large to bring back) unless KEEP_REP=1.
set -u
tag=$1; shift
for spec in "$@"; do
  cfg=${spec%%:*}; layer=${spec#*:}
  out=gpurun_out/${tag}_${layer}
  # the first call of a shape times 4 tail-split candidates x 3 launches before its own launch
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:'spmm_bcsr|spcv_jit' \
    -s ${NCU_SKIP:-17} -c 1 -f -o $out \
    python tools/prof_layer.py --config $cfg --layer $layer --reps 1 --warmup 6 ${PROF_ARGS:-} \
    > $out.ncu.log 2>&1
  echo "$spec rc=$?"
  python tools/ncu_summary.py $out.ncu-rep > $out.summary.txt 2>&1
  ncu -i $out.ncu-rep --page raw --csv > $out.raw.csv 2>/dev/null
  ncu -i $out.ncu-rep --page details > $out.details.txt 2>/dev/null
  ncu -i $out.ncu-rep --page source --csv --print-source sass > $out.sass.csv 2>/dev/null
  [ "${KEEP_REP:-0}" = 1 ] || rm -f $out.ncu-rep
done
