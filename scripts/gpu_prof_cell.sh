#!/bin/bash
# ncu --set full of one product launch of a sweep cell / config ($CFG, launch $SKIP)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python scripts/prof_one.py --config $CFG --evals 1 > gpurun_out/prof_$CFG.log 2>&1 && \
timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:conv_ -s ${SKIP:-4} -c 1 -o /tmp/p python scripts/prof_one.py --config $CFG --evals 1 > gpurun_out/ncu_$CFG.log 2>&1
ncu -i /tmp/p.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$CFG.csv 2>/dev/null
ncu -i /tmp/p.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_$CFG.csv 2>/dev/null
echo done
