for e in "" "SPCV_NWARPS=4" "SPCV_NWARPS=4 SPCV_SPLIT=2" "SPCV_SPLIT=2" "SPCV_TAIL=2" "SPCV_TAIL=4"; do
env $e python tools/prof_layer.py --config c4 --layer b8_project,b12_project,b15_project,b17_project,b15_expand,head --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
done
