#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_lpark.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_lpark.log
TUNE_NPS=1,3 TUNE_OUT=gpurun_out/tune_lpark.json timeout 1800 python scripts/tune_table.py ${CELLS:-qd,sweep_d15_L3,sweep_d15_L4,sweep_d15_L5,sweep_d31_L3,sweep_d31_L4,sweep_d31_L5,sweep_d63_L3,sweep_d63_L4,sweep_d63_L5,sweep_d127_L3,sweep_d127_L4,sweep_d127_L5} > gpurun_out/tune_lpark.log 2>&1
echo done
