#!/bin/bash
# iteration check: all GPU tests, sweep, bench qd
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python scripts/sweep.py --out gpurun_out/sweep.json > gpurun_out/sweep.log 2>&1
for c in qd; do timeout 600 python bench.py --config $c --no-next > gpurun_out/bench_$c.log 2>&1; done
echo done
