for e in "" "SPCV_JIT_STAGES=2" "SPCV_JIT_WARPS=10 SPCV_JIT_STAGES=2" "SPCV_JIT_WARPS=12 SPCV_JIT_STAGES=2" "SPCV_JIT_WARPS=14 SPCV_JIT_STAGES=2" "SPCV_JIT_WARPS=6 SPCV_JIT_STAGES=4" "SPCV_JIT_STAGES=4"; do
env $e python tools/prof_layer.py --config c2-b256 --layer pw2,pw3 --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
done
