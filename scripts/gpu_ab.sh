#!/bin/bash
# A/B of an environment switch on bench lines: VARS="NAME=a NAME=b" CONFIGS="qd dd"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CONFIGS:-qd dd}; do for v in ${VARS:-X=0}; do
  env $v timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/ab_${c}_${v}.log 2>&1
done; done
echo done
