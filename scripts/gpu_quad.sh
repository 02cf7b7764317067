#!/bin/bash
# the quad kernel (MDPS_CONV_KERNEL=3): parity of every default-digit path under it, then A/B timing
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
MDPS_CONV_KERNEL=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_batch.py -q -x > gpurun_out/pytest_quad.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_quad.log
VARS="MDPS_CONV_KERNEL=0 MDPS_CONV_KERNEL=3" CONFIGS="${CONFIGS:-qd sweep_d15_L4 sweep_d31_L4 sweep_d63_L4 sweep_d127_L4 sweep_d15_L5 sweep_d31_L5 sweep_d63_L5 sweep_d127_L5 sweep_d63_L3 sweep_d127_L3 od}" bash scripts/gpu_ab.sh
echo done
