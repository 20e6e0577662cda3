#!/bin/bash
# Round-end evidence on one B200 (outputs under gpurun_out/, TAG prefix).
tag=${1:-r2e}
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu_tests.log 2>&1
python bench.py > gpurun_out/${tag}_bench.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${tag}_reference.log 2>&1
for c in c1 c2-b1; do python bench.py --config $c > gpurun_out/${tag}_bench_$c.log 2>&1; done
for gb in 32 64 128; do python bench.py --global-batch $gb --no-alt > gpurun_out/${tag}_bench_gb$gb.log 2>&1; done
python tools/bench_configs.py --out gpurun_out/${tag}_configs > gpurun_out/${tag}_configs.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 3 > gpurun_out/${tag}_launches.log 2>&1
ncu --profile-from-start off --clock-control none --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed \
    python tools/step_profile.py > gpurun_out/${tag}_step_metrics.csv 2> gpurun_out/${tag}_step_metrics.log
python tools/step_profile.py --traffic gpurun_out/${tag}_step_metrics.csv > gpurun_out/${tag}_traffic.json
tools/ncu_layers.sh ${tag} c2-b256:pw13 c2-b256:pw7 c3:c3_s90_b4
# per-CTA phase timelines (needs make VARIANT=tl VFLAGS=-DSPCV_TIMELINE beforehand)
if [ -f paper_1911_09723_b200/lib/variants/libspcv_cu_tl.so ]; then
  ( export SPCV_CU_LIB=paper_1911_09723_b200/lib/variants/libspcv_cu_tl.so
    python tools/timeline.py --config c2-b256 --layer pw4,pw5,pw7,pw12,pw13
    python tools/timeline.py --config c3 --layer c3_s90_b4,c3_s90_b2,c3_s90_b1
    python tools/timeline.py --config c5 --layer c5_s90,c5_s98
    python tools/timeline.py --config c4 --layer b8_expand,b12_project,b15_expand,head ) > gpurun_out/${tag}_timeline.log 2>&1
fi
