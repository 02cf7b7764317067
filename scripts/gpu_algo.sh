#!/bin/bash
# EFT (algo 1) vs digits (algo 2) on the low-limb cells
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for c in ${CONFIGS:-dd qd sweep_d15_L2 sweep_d63_L2 sweep_d127_L2 sweep_d31_L3 sweep_d63_L3 sweep_d15_L4 sweep_d63_L4}; do for a in 1 2; do
  timeout 600 python bench.py --config $c --algo $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-next > gpurun_out/algo_${c}_$a.log 2>&1
done; done
echo done
