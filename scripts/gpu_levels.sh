#!/bin/bash
# per-launch durations of one evaluation (qd, d15 L4, od) and the executed FP64 instruction counters of one od product launch
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in qd sweep_d15_L4 sweep_d15_L5 od; do
  python scripts/prof_one.py --config $cfg --evals 2 > gpurun_out/lv_$cfg.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,launch__grid_size,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/lv_launches_$cfg.csv python scripts/prof_one.py --config $cfg --evals 2 > /dev/null 2>&1
done
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:conv_ -s 8 -c 1 --csv --log-file gpurun_out/fp64_counts_od.csv python scripts/prof_one.py --config od --evals 1 > /dev/null 2>&1
timeout 600 ncu --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:conv_ -s 0 -c 1 --csv --log-file gpurun_out/fp64_counts_qd.csv python scripts/prof_one.py --config qd --evals 1 > /dev/null 2>&1
echo done
