for img in 32 64; do
  for sm in 1 2; do
    SPCV_SMALL=$sm python tools/prof_layer.py --config c2-b256 --layer pw4,pw5,pw6,pw7,pw12,pw13 --images $img --reps 7 --check 1 2>&1 | grep -E "median|MISM" | sed -E "s/^/[img=$img small=$sm] /"
  done
done
