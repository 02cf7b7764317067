#!/bin/bash
# per-launch durations of one evaluation (qd, d15 L4/L5, d31 L4)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in qd sweep_d15_L4 sweep_d15_L5 sweep_d31_L4; do
  python scripts/prof_one.py --config $cfg --evals 2 > gpurun_out/lv2_$cfg.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/lv2_launches_$cfg.csv python scripts/prof_one.py --config $cfg --evals 2 > /dev/null 2>&1
done
echo done
