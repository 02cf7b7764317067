#!/bin/bash
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_fuzz.py tests/test_gpu_solve.py tests/test_gpu_newton.py -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_pdl.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_pdl.log
timeout 900 python scripts/pdl_ab.py > gpurun_out/pdl_ab.jsonl 2> gpurun_out/pdl_ab.err
timeout 900 python scripts/sweep.py --l2-both --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
echo done
