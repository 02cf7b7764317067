#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in sweep_d63_L8 sweep_d63_L10; do
python scripts/prof_one.py --config $c --evals 2 > gpurun_out/prof_plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:accum_dig -s 1 -c 1 -o gpurun_out/prof_accum_$c python scripts/prof_one.py --config $c --evals 2 > gpurun_out/ncu_accum_$c.log 2>&1
done
