#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TUNE_NPS=1,3 TUNE_OUT=gpurun_out/tune_l2.json timeout 900 python scripts/tune_table.py sweep_d15_L2,sweep_d31_L2,sweep_d63_L2,sweep_d127_L2 > gpurun_out/tune_l2.log 2>&1
echo done
