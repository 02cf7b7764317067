#!/bin/bash
# fused-parts kernel: geometry + parity tests, then the (F, P, NP) table on the L <= 5 cells
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fused.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fused.log
TUNE_OUT=gpurun_out/tune_fused.json timeout 1800 python scripts/tune_table.py ${CELLS:-qd,sweep_d15_L3,sweep_d15_L4,sweep_d15_L5,sweep_d31_L3,sweep_d31_L4,sweep_d31_L5,sweep_d63_L3,sweep_d63_L4,sweep_d63_L5,sweep_d127_L3,sweep_d127_L4,sweep_d127_L5,sweep_d15_L2,sweep_d31_L2,sweep_d63_L2,sweep_d127_L2} > gpurun_out/tune_fused.log 2>&1
echo done
