for e in "" "SPCV_STEPS=4" "SPCV_STEPS=4 SPCV_REGCAP=0"; do
env $e python tools/prof_layer.py --config c2-b256 --layer pw4,pw5,pw6,pw7 --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
env $e python tools/prof_layer.py --config c3 --layer c3_s90_b1,c3_s70_b1 --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
env $e python tools/prof_layer.py --config c4 --layer b8_expand,b12_expand --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
done
