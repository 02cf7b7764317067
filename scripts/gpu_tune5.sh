#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_t5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t5.log
TUNE_OUT=gpurun_out/tune5.json timeout 1800 python scripts/tune_table.py ${CELLS} > gpurun_out/tune5.log 2>&1
echo done
