#!/bin/bash
# solver evidence: launch list of the solve bench (qd, od, deca) and ncu --set full
# of the persistent solver kernel and the Gauss-Jordan kernel (od, deca)
cd $GRAFT_REPO_ROOT
python scripts/bench_solve.py qd od deca --trace > gpurun_out/bench_solve_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_solve.csv python scripts/bench_solve.py qd od deca > gpurun_out/ncu_solve_launch.log 2>&1
for c in od deca; do
ncu --set full --clock-control none --import-source on -k regex:"ts_main" -c 1 -o gpurun_out/prof_solve_$c python scripts/bench_solve.py $c > gpurun_out/ncu_full_solve_$c.log 2>&1
done
echo done
