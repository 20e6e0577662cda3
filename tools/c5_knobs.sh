for l in c5_s98 c5_s95 c5_s90; do
for e in "" "SPCV_STEPS=2" "SPCV_NF=2" "SPCV_NF=2 SPCV_STEPS=2" "SPCV_NWARPS=8"; do
env $e python tools/prof_layer.py --config c5 --layer $l --reps 5 --warmup 2 --check 1 2>&1 | grep -E "median|Error" | sed "s/^/[$e] /; s/(prep.*slots=[0-9]*//"
done; done
