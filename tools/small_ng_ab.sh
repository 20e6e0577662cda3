for round in 1 2; do for v in main ng16 ng4; do
  if [ $v = main ]; then L=paper_1911_09723_b200/lib/libspcv_cu.so; else L=paper_1911_09723_b200/lib/variants/libspcv_cu_$v.so; fi
  for c in c1 c2-b1; do
  SPCV_CU_LIB=$L python bench.py --config $c 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$round $v $c', d['ms_per_step'], d['timing']['median_step_ms'], 'graph', d['graph']['ms_per_step'], 'net b1', d['network']['batch1_latency_ms'])"
  done
done; done
