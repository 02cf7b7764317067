#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_tail.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_tail.log
timeout 900 python scripts/pdl_ab.py qd,sweep_d15_L3,sweep_d15_L4,sweep_d15_L5,sweep_d31_L4,sweep_d31_L5,sweep_d63_L4,sweep_d63_L3 > gpurun_out/tail_ab.jsonl 2> gpurun_out/tail_ab.err
echo done
