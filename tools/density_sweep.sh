# steady state without a tail: 2960 images of 4x4 = 1480 tiles of 32 columns = 10 per SM
for bh in 4 1; do for s in 0.9 0.7; do for p in 0 2; do
SPCV_PERSIST=$p python tools/prof_layer.py --adhoc 512,512,4,4,$s,$bh,2960 --reps 5 --warmup 2 --check 1 2>&1 | grep -E "median|Error" | sed "s/^/[bh=$bh s=$s persist=$p] /; s/(prep.*slots=[0-9]*//"
done; done; done
