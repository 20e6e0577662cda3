for e in "" "SPCV_TILE_T=64" "SPCV_TILE_T=64 SPCV_NWARPS=4" "SPCV_NWARPS=4" "SPCV_TILE_T=32" "SPCV_TILE_T=32 SPCV_NWARPS=4"; do
env $e python tools/prof_layer.py --config c2-b256 --layer pw4,pw5,pw6 --reps 7 --warmup 3 --check 1 2>&1 | grep -E "median|Error|MISMATCH" | sed "s/(prep.*slots=[0-9]*//; s/(alg.*//; s/^/[$e] /"
done
