#!/bin/bash
# all GPU tests (stop at the first failure) and the sweep
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_fs.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_fs.log
timeout 900 python scripts/sweep.py --out gpurun_out/sweep_fs.json > gpurun_out/sweep_fs.log 2>&1
echo done
