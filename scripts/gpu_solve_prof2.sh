#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/solve_trace.py od > gpurun_out/solve_trace.log 2>&1
python scripts/prof_solve.py od > gpurun_out/prof_solve.log 2>&1 && \
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:ts_main -c 1 -o /tmp/ps python scripts/prof_solve.py od > gpurun_out/ncu_solve.log 2>&1
ncu -i /tmp/ps.ncu-rep --page raw --csv > gpurun_out/ncu_raw_solve.csv 2>/dev/null
ncu -i /tmp/ps.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_solve.csv 2>/dev/null
echo done
