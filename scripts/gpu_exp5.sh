#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TUNE_NPS=3,4 TUNE_OUT=gpurun_out/tune_cap128.json timeout 1800 python scripts/tune_table.py ${CELLS:-qd,sweep_d15_L4,sweep_d31_L4,sweep_d63_L4,sweep_d15_L5,sweep_d31_L5,sweep_d63_L5} > gpurun_out/tune_cap128.log 2>&1
timeout 900 python scripts/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_geometry.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_exp5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_exp5.log
echo done
