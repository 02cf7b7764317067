#!/bin/bash
# NB (double-buffered persistent blocks): geometry/parity tests + tune table on the digit cells
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_t4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_t4.log
TUNE_OUT=gpurun_out/tune4.json timeout 2400 python scripts/tune_table.py qd,od,deca,sweep_d15_L3,sweep_d15_L4,sweep_d15_L5,sweep_d15_L8,sweep_d15_L10,sweep_d31_L3,sweep_d31_L4,sweep_d31_L5,sweep_d31_L8,sweep_d31_L10,sweep_d63_L3,sweep_d63_L4,sweep_d63_L5,sweep_d63_L8,sweep_d63_L10,sweep_d127_L3,sweep_d127_L4,sweep_d127_L5,sweep_d127_L8,sweep_d127_L10 > gpurun_out/tune4.log 2>&1
echo done
