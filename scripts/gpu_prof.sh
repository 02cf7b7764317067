#!/bin/bash
cd $GRAFT_REPO_ROOT
for c in ${PCONFIGS:-od deca}; do
python scripts/prof_one.py --config $c --evals 2 > gpurun_out/prof_plain_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-conv_} -s ${SKIP:-24} -c 1 -o gpurun_out/prof_conv_$c python scripts/prof_one.py --config $c --evals 2 > gpurun_out/ncu_full_$c.log 2>&1
done
echo done
