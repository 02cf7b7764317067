#!/bin/bash
# quick iteration: product-kernel tests + sweep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_geometry.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge.py tests/test_gpu_real.py -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_iter5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_iter5.log
timeout 900 python scripts/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
echo done
