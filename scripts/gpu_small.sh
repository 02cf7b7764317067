#!/bin/bash
# small-D diagnosis: per-launch durations (grid, block) and one full capture per config
cd $GRAFT_REPO_ROOT
for c in ${PCONFIGS:-qd sweep_d15_L8 sweep_d31_L4}; do
python scripts/prof_one.py --config $c --evals 2 > gpurun_out/prof_plain_$c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_$c.csv python scripts/prof_one.py --config $c --evals 2 > gpurun_out/ncu_launch_$c.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv_ -s ${SKIP:-4} -c 1 -o gpurun_out/prof_conv_$c python scripts/prof_one.py --config $c --evals 2 > gpurun_out/ncu_full_$c.log 2>&1
done
echo done
